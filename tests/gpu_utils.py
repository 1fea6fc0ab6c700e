"""Run the CUDA path through the C ABI and bring every output back to numpy."""
import numpy as np
import torch

import oracle


def to_dev(field):
    from paper_2602_15355_b200 import Gaussians
    return Gaussians(torch.from_numpy(np.ascontiguousarray(field.planes)).cuda(), field.sh_degree)


def to_dev_lod(lod):
    from paper_2602_15355_b200 import Lod
    if lod is None:
        return None
    return Lod(torch.from_numpy(np.ascontiguousarray(lod.tile_level)).cuda(), lod.levels, lod.delta, lod.thresholds)


def gpu_batch(ctx, field, cams, images=True, want_unsorted=True, want_keys=True, want_gray=False, lod=None):
    """One batch (len(cams) <= 64, same W,H) through K1..K7; numpy outputs."""
    from paper_2602_15355_b200 import gsr
    G = to_dev(field)
    V, n = len(cams), field.n
    W, H = int(cams[0]["width"]), int(cams[0]["height"])
    gx, gy = (W + 15) // 16, (H + 15) // 16
    T = V * gx * gy
    rec = torch.full((V, max(n, 1), 12), float("nan"), dtype=torch.float32, device="cuda")
    binr = torch.full((10 * V * max(n, 1),), -1, dtype=torch.int32, device="cuda")
    gsr.gsr_project(ctx, G, cams, rec, binr, lod=to_dev_lod(lod))
    cap = 0
    vals = torch.empty(1, dtype=torch.int32, device="cuda")
    ranges = torch.full((T, 2), -1, dtype=torch.int32, device="cuda")
    try:
        gsr.gsr_bin_sort(ctx, binr, n, cams, vals, 0, ranges)
        K = 0
    except gsr.GsrError as e:
        assert e.status == gsr.GSR_ECAPACITY
        K = e.required
    cap = max(K, 1)
    vals = torch.full((cap,), -1, dtype=torch.int32, device="cuda")
    keys = torch.full((cap,), -1, dtype=torch.int64, device="cuda") if want_keys else None
    ku = torch.full((cap,), -1, dtype=torch.int64, device="cuda") if want_unsorted else None
    vu = torch.full((cap,), -1, dtype=torch.int32, device="cuda") if want_unsorted else None
    K2 = gsr.gsr_bin_sort(ctx, binr, n, cams, vals, cap, ranges, keys=keys, keys_unsorted=ku, vals_unsorted=vu)
    assert K2 == K
    partial = torch.full((T,), float("nan"), dtype=torch.float32, device="cuda")
    rgbu = torch.full((V, H, W, 4), float("nan"), dtype=torch.float32, device="cuda") if images else None
    tf = torch.full((V, H, W), float("nan"), dtype=torch.float32, device="cuda") if images else None
    nc = torch.full((V, H, W), -1, dtype=torch.int32, device="cuda") if images else None
    nfrag = torch.zeros(2, dtype=torch.int64, device="cuda")
    gray = torch.full((V, H, W), float("nan"), dtype=torch.float32, device="cuda") if want_gray else None
    gsr.gsr_composite(ctx, rec, n, vals, ranges, cams, partial, rgbu=rgbu, t_final=tf, n_contrib=nc, n_frag=nfrag,
                      gray=gray)
    scores = torch.full((V,), float("nan"), dtype=torch.float32, device="cuda")
    gsr.gsr_score_views(ctx, partial, cams, scores)
    torch.cuda.synchronize()
    b = binr.cpu().numpy().view(np.uint32)
    M = V * max(n, 1)
    out = dict(K=K, rec=rec.cpu().numpy(), span=b[:8 * M].reshape(V, max(n, 1), 8),
               depth=b[8 * M:9 * M].reshape(V, max(n, 1)), n_tiles=b[9 * M:].reshape(V, max(n, 1)),
               vals=vals.cpu().numpy().view(np.uint32)[:K], ranges=ranges.cpu().numpy().view(np.uint32),
               partial=partial.cpu().numpy(), scores=scores.cpu().numpy(), n_frag=int(nfrag[0].item()),
               n_eval=int(nfrag[1].item()))
    if want_keys:
        out["keys"] = keys.cpu().numpy().view(np.uint64)[:K]
    if want_unsorted:
        out["keys_unsorted"] = ku.cpu().numpy().view(np.uint64)[:K]
        out["vals_unsorted"] = vu.cpu().numpy().view(np.uint32)[:K]
    if want_gray:
        out["gray"] = gray.cpu().numpy()
    if images:
        out.update(rgbu=rgbu.cpu().numpy(), t_final=tf.cpu().numpy(), n_contrib=nc.cpu().numpy().view(np.uint32))
    return out


def oracle_batch(field, cams, images=True, lod=None):
    """The oracle's expected outputs for the same batch."""
    projs = [oracle.project(field, c, lod) for c in cams]
    bs = oracle.bin_sort_batch(projs, cams)
    gx, gy = oracle.grid(cams[0])
    tpv = gx * gy
    res = dict(projs=projs, **bs)
    if images:
        imgs, tfs, ncs, scores, nfrag, neval = [], [], [], [], 0, 0
        for v, (p, c) in enumerate(zip(projs, cams)):
            rv = bs["ranges"][v * tpv:(v + 1) * tpv]
            o = oracle.composite_tiled(p, bs["vals"], rv, c)
            imgs.append(o["rgbu"])
            tfs.append(o["t_final"])
            ncs.append(o["n_contrib"])
            scores.append(o["score"])
            nfrag += o["n_frag"]
            neval += o["n_eval"]
        res.update(rgbu=np.stack(imgs), t_final=np.stack(tfs), n_contrib=np.stack(ncs),
                   scores=np.array(scores), n_frag=nfrag, n_eval=neval)
    return res


def check_projection(gpu, orc, n):
    """Bin records (depth, n_tiles, span records) bit-exact; render records
    bit-exact where visible."""
    for v, p in enumerate(orc["projs"]):
        assert np.array_equal(gpu["n_tiles"][v, :n], p["n_tiles"]), f"view {v}: n_tiles"
        assert np.array_equal(gpu["depth"][v, :n], p["depth_bits"]), f"view {v}: depth"
        vis = p["n_tiles"] > 0
        sp = gpu["span"][v, :n][vis]
        for col, name in [(0, "u"), (1, "v"), (2, "sp_p"), (3, "sp_h"), (4, "sp_ic"), (5, "sp_dys")]:
            assert np.array_equal(sp[:, col], p[name][vis].view(np.uint32)), f"view {v}: span {name}"
        assert np.array_equal(sp[:, 6] & 0xFFFF, p["py0"][vis]) and np.array_equal(sp[:, 6] >> 16, p["py1"][vis])
        assert np.array_equal(sp[:, 7], p["n_tiles"][vis]), f"view {v}: span n_tiles"
        r = gpu["rec"][v, :n][vis]
        for col, name in [(0, "u"), (1, "v"), (2, "A"), (3, "B"), (4, "C"), (5, "o"), (6, "unc"),
                          (8, "r"), (9, "g"), (10, "b")]:
            assert np.array_equal(r[:, col].view(np.uint32), p[name][vis].view(np.uint32)), f"view {v}: {name}"


def gpu_forward_backward(ctx, field, cams, G, lod=None):
    """Forward (K1..K6 with images) + NEXT-3 backward of one batch through the
    C ABI; G [V][H][W][4] upstream gradient -> (rgbu, grads [P][n][4])."""
    from paper_2602_15355_b200 import gsr
    Gd = to_dev(field)
    L = to_dev_lod(lod)
    V, n = len(cams), field.n
    W, H = int(cams[0]["width"]), int(cams[0]["height"])
    T = V * ((W + 15) // 16) * ((H + 15) // 16)
    rec = torch.zeros((V, max(n, 1), 12), dtype=torch.float32, device="cuda")
    binr = torch.zeros((10 * V * max(n, 1),), dtype=torch.int32, device="cuda")
    gsr.gsr_project(ctx, Gd, cams, rec, binr, lod=L)
    ranges = torch.zeros((T, 2), dtype=torch.int32, device="cuda")
    vals = torch.zeros(1, dtype=torch.int32, device="cuda")
    try:
        K = gsr.gsr_bin_sort(ctx, binr, n, cams, vals, 0, ranges)
    except gsr.GsrError as e:
        K = e.required
    vals = torch.zeros(max(K, 1), dtype=torch.int32, device="cuda")
    gsr.gsr_bin_sort(ctx, binr, n, cams, vals, max(K, 1), ranges)
    partial = torch.zeros(T, dtype=torch.float32, device="cuda")
    rgbu = torch.zeros((V, H, W, 4), dtype=torch.float32, device="cuda")
    gsr.gsr_composite(ctx, rec, n, vals, ranges, cams, partial, rgbu=rgbu)
    dG = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    grads = torch.zeros_like(Gd.planes)
    gsr.gsr_backward(ctx, Gd, cams, rec, binr, vals, ranges, rgbu, dG, grads, lod=L)
    torch.cuda.synchronize()
    return rgbu.cpu().numpy(), grads.cpu().numpy()
