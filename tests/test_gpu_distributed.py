"""The N > 1 path with the real CUDA scorer (VERDICT r1 "missing" 1-2): two
ranks on the one B200, gloo process group (host-mediated collectives; the
ranks' kernels never wait on each other), each running libgsr through
ViewScorer.  SURVEY.md §8(e): C1 broadcast of the packed field from rank 0,
strided view ownership, C2 all-gather + un-stride, K8 on every rank; the
config-5 coarse -> top-k -> fine flow.  Per-view computation does not depend
on P, so every rank's scores must be bit-identical to the single-process
run of the same scorer, with the same NBV and top-k."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    sc = synth.make_scene(2, n_override=20000, views=24)  # terrain tile, SH 3
    cams = synth.with_resolution(sc.cameras, 160, 128, 160.0)
    return sc, cams


def _fine(c):
    return synth.with_resolution(c, 320, 256, 320.0)


def _scorer(planes, sh_degree):
    from paper_2602_15355_b200 import Gaussians
    from paper_2602_15355_b200.pipeline import ViewScorer
    return ViewScorer(Gaussians(planes, sh_degree), batch_views=8, n_slots=2)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2602_15355_b200 import distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc, cams = _scene()
        planes = torch.zeros(sc.field.planes.shape, dtype=torch.float32, device="cuda")
        if rank == 0:
            planes.copy_(torch.from_numpy(sc.field.planes))
        D.broadcast_field(planes)  # C1: only rank 0 holds the field before this
        torch.cuda.synchronize()
        digest = hashlib.sha256(planes.cpu().numpy().tobytes()).hexdigest()
        s = _scorer(planes, sc.field.sh_degree)
        score = s.score_views
        select = s.select
        scores, sel = D.score_and_select(cams, score, select, k=5)
        cs, top, fs, nbv = D.hierarchical_select(cams, _fine, score, score, select, top_k=6)
        q.put((rank, digest, scores.cpu().numpy(), sel.cpu().numpy().tolist(), cs.cpu().numpy(), top.tolist(),
               fs.cpu().numpy(), nbv))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_ranks_broadcast_score_gather_select_on_gpu():
    import torch.multiprocessing as mp
    sc, cams = _scene()
    # single-process run of the same scorer (the P = 1 result)
    planes = torch.from_numpy(sc.field.planes).cuda()
    s = _scorer(planes, sc.field.sh_degree)
    ref = s.score_views(cams).cpu().numpy()
    ref_sel = s.select(torch.from_numpy(ref).cuda(), 5).cpu().numpy().tolist()
    top = s.select(torch.from_numpy(ref).cuda(), 6).cpu().numpy().astype(np.int64)
    fref = s.score_views(_fine(cams[top])).cpu().numpy()
    best = int(top[int(np.argmax(fref))])
    want_digest = hashlib.sha256(sc.field.planes.tobytes()).hexdigest()
    torch.cuda.synchronize()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, digest, scores, sel, cs, t, fs, nbv in res:
        assert digest == want_digest, rank  # the field bytes arrived intact
        assert np.array_equal(scores, ref), rank  # bit-identical to P = 1
        assert sel == ref_sel, rank
        assert np.array_equal(cs, ref) and t == top.tolist(), rank
        assert np.array_equal(fs, fref) and nbv == best, rank
