"""Host orchestration of one scoring pass (Alg. 1 L147-154 body): for every
candidate view, K1 project -> K2..K5 bin+sort -> K6 composite -> K7 score,
batched by view; then K8 top-k.  All arithmetic runs in libgsr's kernels;
this file only sizes buffers and sequences the C-ABI calls on one stream.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import gsr
from .gsr import CAM_DTYPE, Context, Gaussians, GsrError


def tiles_per_view(cam) -> int:
    W, H = int(cam["width"]), int(cam["height"])
    return ((W + 15) // 16) * ((H + 15) // 16)


@dataclass
class BatchOut:
    n_keys: int
    images: Optional[torch.Tensor] = None  # [V][H][W][4]


class ViewScorer:
    """Scores candidate views of one Gaussian field on one GPU.

    ``batch_views`` views share one K1 launch (the parameter planes are read
    once per batch) and one pair of sorts.  Buffers grow on demand; the key
    capacity follows the capacity protocol of gsr_bin_sort (GSR_ECAPACITY
    returns the required size, we grow by 25% and retry)."""

    def __init__(self, field: Gaussians, batch_views: int = 8, ctx: Optional[Context] = None,
                 stream: Optional[torch.cuda.Stream] = None):
        self.field = field
        self.dev = field.planes.device
        self.ctx = ctx or Context(self.dev.index or 0)
        self.V = min(int(batch_views), gsr.GSR_MAX_VIEWS)
        self.stream = stream
        n = field.n
        self.rec = torch.empty((self.V, max(n, 1), 12), dtype=torch.float32, device=self.dev)
        self.bin = torch.empty((4, self.V, max(n, 1)), dtype=torch.int32, device=self.dev)
        self.capacity = 0
        self.vals = None
        self.keys = None
        self.ranges = None
        self.partial = None
        self.n_frag = torch.zeros(2, dtype=torch.int64, device=self.dev)  # [blended, evaluated]
        self.last_keys = []

    def _ensure_keys(self, cap: int, want_keys: bool):
        if cap > self.capacity or (want_keys and self.keys is None):
            self.capacity = max(cap, self.capacity)
            self.vals = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=self.dev)
            self.keys = torch.empty(max(self.capacity, 1), dtype=torch.int64, device=self.dev) if want_keys else None

    def _ensure_tiles(self, T: int):
        if self.ranges is None or self.ranges.shape[0] < T:
            self.ranges = torch.empty((T, 2), dtype=torch.int32, device=self.dev)
            self.partial = torch.empty(T, dtype=torch.float32, device=self.dev)

    def run_batch(self, cams: np.ndarray, scores_out: torch.Tensor, images: Optional[torch.Tensor] = None,
                  t_final=None, n_contrib=None, want_keys: bool = False) -> BatchOut:
        """Score len(cams) <= batch_views same-resolution views into scores_out[0:len(cams)]."""
        cams = gsr.cams_array(cams)
        V = len(cams)
        assert 0 < V <= self.V
        n = self.field.n
        tpv = tiles_per_view(cams[0])
        self._ensure_tiles(V * tpv)
        if self.capacity == 0:
            self._ensure_keys(max(1 << 20, 4 * n * V), want_keys)
        elif want_keys:
            self._ensure_keys(self.capacity, True)
        st = self.stream
        gsr.gsr_project(self.ctx, self.field, cams, self.rec, self.bin, st)
        # rec / bin hold [V][n][12] and [4][V][n] for THIS batch's V, packed from the
        # start of the (batch_views-sized) buffers: pass the base pointers.
        while True:
            try:
                K = gsr.gsr_bin_sort(self.ctx, self.bin, n, cams, self.vals, self.capacity, self.ranges,
                                     keys=self.keys if want_keys else None, stream=st)
                break
            except GsrError as e:
                if e.status != gsr.GSR_ECAPACITY:
                    raise
                self._ensure_keys(int(math.ceil(e.required * 1.25)) + 1024, want_keys)
        gsr.gsr_composite(self.ctx, self.rec, n, self.vals, self.ranges, cams, self.partial, rgbu=images,
                          t_final=t_final, n_contrib=n_contrib, n_frag=self.n_frag, stream=st)
        gsr.gsr_score_views(self.ctx, self.partial, cams, scores_out, st)
        return BatchOut(K, images)

    def score_views(self, cams: np.ndarray, scores_out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Scores for all of ``cams`` (any count; same resolution), batched."""
        cams = gsr.cams_array(cams)
        if scores_out is None:
            scores_out = torch.empty(len(cams), dtype=torch.float32, device=self.dev)
        self.last_keys = []
        for b0 in range(0, len(cams), self.V):
            b1 = min(len(cams), b0 + self.V)
            out = self.run_batch(cams[b0:b1], scores_out[b0:b1])
            self.last_keys.append(out.n_keys)
        return scores_out

    def select(self, scores: torch.Tensor, k: int = 1, exclude=None) -> torch.Tensor:
        out = torch.empty(k, dtype=torch.int32, device=self.dev)
        gsr.gsr_select_nbv(self.ctx, scores, k, out, exclude, self.stream)
        return out
