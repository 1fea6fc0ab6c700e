"""Multi-process (gloo, CPU) tests of the data-parallel driver's host logic:
strided view ownership, all-gather + un-striding, top-k on every rank, the
config-5 hierarchical coarse -> top-k -> fine flow.  The
per-view scorer is a test-only stand-in (the CPU oracle); the product path
scores with libgsr on the GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2602_15355_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_scorer(field):
    def score(cams):
        sc, _, _, _ = oracle.render_views(field, cams, n_threads=1)
        return torch.tensor(sc, dtype=torch.float32)
    return score


def _select(scores, k, exclude):
    return torch.tensor(oracle.select_topk(scores.numpy(), k, exclude), dtype=torch.int32)


def _worker(rank, world, port, out_q, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = synth.make_scene(1, n_override=1500, views=10)
        cams = synth.with_resolution(sc.cameras, 48, 48, 48.0)
        if mode == "bcast":
            # C1: rank 0 holds the packed field, the others start from zeros
            planes = torch.from_numpy(sc.field.planes.copy()) if rank == 0 else torch.zeros(sc.field.planes.shape)
            D.broadcast_field(planes)
            fld = synth.GaussianField(planes.numpy(), sc.field.sh_degree)
            scores, sel = D.score_and_select(cams, _oracle_scorer(fld), _select, k=3)
            out_q.put((rank, planes.numpy().tobytes() == sc.field.planes.tobytes(), scores.numpy().tolist(),
                       sel.numpy().tolist()))
        elif mode == "flat":
            scores, sel = D.score_and_select(cams, _oracle_scorer(sc.field), _select, k=3)
            out_q.put((rank, scores.numpy().tolist(), sel.numpy().tolist()))
        else:
            fine = lambda c: synth.with_resolution(c, 96, 96, 96.0)  # noqa: E731
            cs, top, fs, nbv = D.hierarchical_select(cams, fine, _oracle_scorer(sc.field), _oracle_scorer(sc.field),
                                                     _select, top_k=4)
            out_q.put((rank, cs.numpy().tolist(), top.tolist(), fs.numpy().tolist(), nbv))
    finally:
        dist.destroy_process_group()


def _run(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


def test_shard_and_unstride_are_inverse():
    for n in (1, 7, 16, 1024):
        for P in (1, 2, 3, 8):
            L = D.shard_len(n, P)
            g = torch.full((P, L), -1.0)
            for r in range(P):
                idx = D.shard_indices(n, r, P)
                g[r, :len(idx)] = torch.tensor(idx, dtype=torch.float32)
            assert D.unstride(g, n).tolist() == list(range(n))


def _reference():
    sc = synth.make_scene(1, n_override=1500, views=10)
    cams = synth.with_resolution(sc.cameras, 48, 48, 48.0)
    ref, _, _, _ = oracle.render_views(sc.field, cams, n_threads=1)
    return sc, cams, ref


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_score_gather_select(world):
    """Every rank ends with the full score vector in view order (identical to
    the single-process scores, so independent of P) and the same top-k."""
    sc, cams, ref = _reference()
    res = _run(world, "flat")
    exp_sel = oracle.select_topk(np.float32(ref), 3).tolist()
    for rank, scores, sel in res:
        assert np.array_equal(np.float32(scores), np.float32(ref)), rank
        assert sel == exp_sel


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_broadcast_field_then_score(world):
    """C1: after broadcast_field every rank holds rank 0's field bytes, and
    scoring from the broadcast copies reproduces the single-process scores."""
    sc, cams, ref = _reference()
    res = _run(world, "bcast")
    exp_sel = oracle.select_topk(np.float32(ref), 3).tolist()
    for rank, same, scores, sel in res:
        assert same, rank
        assert np.array_equal(np.float32(scores), np.float32(ref)), rank
        assert sel == exp_sel


def test_gloo_hierarchical_coarse_to_fine():
    """Config-5 flow: coarse scores gathered, top-4 on every rank, fine pass
    re-rendered at 2x resolution, argmax mapped back to a coarse index."""
    sc, cams, ref = _reference()
    res = _run(2, "hier")
    top = oracle.select_topk(np.float32(ref), 4)
    fine = synth.with_resolution(cams[top], 96, 96, 96.0)
    fref, _, _, _ = oracle.render_views(sc.field, fine, n_threads=1)
    best = int(top[oracle.select_topk(np.float32(fref), 1)[0]])
    for rank, cs, t, fs, nbv in res:
        assert t == top.tolist() and nbv == best
        assert np.array_equal(np.float32(fs), np.float32(fref))
