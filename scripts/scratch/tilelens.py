import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_2602_15355_b200 import Context, gsr, Gaussians
from tests.gpu_utils import to_dev
for cfg, views in ((3, [0, 200, 500, 900]), (4, [0, 21, 42, 63])):
    sc = synth.make_scene(cfg)
    G = to_dev(sc.field)
    ctx = Context(0)
    cams = sc.cameras[views]
    V, n = len(cams), sc.field.n
    W, H = int(cams[0]["width"]), int(cams[0]["height"])
    T = V * ((W + 15) // 16) * ((H + 15) // 16)
    rec = torch.empty((V, n, 12), device="cuda"); binr = torch.empty(10 * V * n, dtype=torch.int32, device="cuda")
    gsr.gsr_project(ctx, G, cams, rec, binr)
    ranges = torch.empty((T, 2), dtype=torch.int32, device="cuda")
    vals = torch.empty(1, dtype=torch.int32, device="cuda")
    try:
        gsr.gsr_bin_sort(ctx, binr, n, cams, vals, 0, ranges); K = 0
    except gsr.GsrError as e:
        K = e.required
    vals = torch.empty(K, dtype=torch.int32, device="cuda")
    gsr.gsr_bin_sort(ctx, binr, n, cams, vals, K, ranges)
    r = ranges.cpu().numpy().astype(np.int64)
    L = r[:, 1] - r[:, 0]
    nt = binr.cpu().numpy()[9 * V * n:]
    print(f"c{cfg}: K/view {K/V:.0f} visible/view {(nt>0).sum()/V:.0f} tiles {T} len mean {L.mean():.0f} p50 {np.median(L):.0f} p99 {np.percentile(L,99):.0f} max {L.max()} >4K {(L>4096).sum()} >8K {(L>8192).sum()} >16K {(L>16384).sum()}")
