"""Multi-GPU scoring over one node: data parallel over candidate views.

SURVEY.md §8(e): (1) broadcast the packed Gaussian planes from rank 0 (one
NCCL broadcast per field revision, NVLink/NVSwitch); (2) strided ownership,
view v belongs to rank v mod P (the Fibonacci index correlates with
elevation, so contiguous slices would be load-imbalanced); (3) each rank
renders and scores its views (libgsr K1..K7); (4) one all_gather_into_tensor
of the padded [P][ceil(N/P)] scores, un-strided back to view order; (5) K8
top-k on every rank with the deterministic tie rule, so all ranks agree
without a further broadcast.  Per-view computation does not depend on P, so
scores are bit-identical across P.

The collective plumbing is torch.distributed (NCCL on GPUs; gloo for the
CPU tests of this host logic).  The scorer / selector are injected so the
same orchestration is exercised by CPU tests with a test-only scorer.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


def shard_indices(n_views: int, rank: int, world: int) -> np.ndarray:
    """Views owned by `rank`: v = rank, rank + P, rank + 2P, ..."""
    return np.arange(rank, n_views, world, dtype=np.int64)


def shard_len(n_views: int, world: int) -> int:
    return (n_views + world - 1) // world


def unstride(gathered: torch.Tensor, n_views: int) -> torch.Tensor:
    """[P][L] per-rank strided scores -> [n_views] in view order:
    full[v] = gathered[v % P][v // P]."""
    P, L = gathered.shape
    return gathered.t().reshape(P * L)[:n_views]


def broadcast_field(planes: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """C1: replicate the contiguous packed planes from `src` (in place)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(planes, src=src, group=group)
    return planes


def gather_scores(local: torch.Tensor, n_views: int, group=None) -> torch.Tensor:
    """C2: all-gather each rank's padded strided scores, return [n_views]."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local[:n_views]
    L = shard_len(n_views, world)
    pad = torch.zeros(L, dtype=local.dtype, device=local.device)
    pad[: local.numel()] = local
    out = torch.empty((world, L), dtype=local.dtype, device=local.device)
    try:
        dist.all_gather_into_tensor(out, pad, group=group)
    except (RuntimeError, NotImplementedError):  # backends without the fused op
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        out = torch.stack(parts)
    return unstride(out, n_views)


def score_and_select(cams: np.ndarray, score_fn: Callable[[np.ndarray], torch.Tensor],
                     select_fn: Callable[[torch.Tensor, int, Optional[np.ndarray]], torch.Tensor],
                     k: int = 1, exclude: Optional[np.ndarray] = None, group=None):
    """One Alg. 1 scoring iteration (L147-154) on this rank: score the owned
    views, all-gather, select top-k.  Returns (scores [N], selected [k])."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mine = shard_indices(len(cams), rank, world)
    local = score_fn(cams[mine]) if len(mine) else None
    if local is None:
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
        local = torch.zeros(0, dtype=torch.float32, device=dev)
    scores = gather_scores(local, len(cams), group)
    return scores, select_fn(scores, k, exclude)


def hierarchical_select(coarse_cams: np.ndarray, fine_cams_fn: Callable[[np.ndarray], np.ndarray],
                        coarse_score_fn, fine_score_fn, select_fn, top_k: int = 64, group=None):
    """Config 5 (SURVEY §8(c) reading "Top-k in config 5"): coarse pass over all
    candidates, gather, top-k, fine pass re-rendering those k views at the fine
    resolution (sharded again), gather, argmax.  Returns (coarse scores, top-k
    indices, fine scores, NBV index into coarse_cams)."""
    cs, top = score_and_select(coarse_cams, coarse_score_fn, select_fn, top_k, None, group)
    top_np = top.detach().cpu().numpy().astype(np.int64)
    fine = fine_cams_fn(coarse_cams[top_np])
    fs, best = score_and_select(fine, fine_score_fn, select_fn, 1, None, group)
    return cs, top_np, fs, int(top_np[int(best.reshape(-1)[0].item())])
