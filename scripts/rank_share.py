"""Per-rank workload of the N-GPU bench emulated on one GPU: score 1024 / N
strided c3 views per pass with different batch sizes (device time per pass)."""
import sys
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_15355_b200 import Gaussians  # noqa: E402
from paper_2602_15355_b200.pipeline import ViewScorer  # noqa: E402

sc = synth.make_scene(3)
G = Gaussians(torch.from_numpy(sc.field.planes).cuda(), 3)
for N in (1, 2, 4, 8):
    cams = sc.cameras[0::N]
    for b in (16, 32):
        s = ViewScorer(G, batch_views=b)
        for _ in range(2):
            s.score_views(cams)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            s.score_views(cams)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"N={N} views/rank={len(cams)} batch={b}: {ms:.2f} ms/pass -> {len(cams) / ms * 1e3 * N:.0f} views/s at N")
        del s
        torch.cuda.empty_cache()
