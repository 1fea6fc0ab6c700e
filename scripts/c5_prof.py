"""One config-5 coarse pass (4,096 views at 256^2, 2M Gaussians) for ncu launch lists."""
import sys
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_15355_b200 import Gaussians  # noqa: E402
from paper_2602_15355_b200.pipeline import ViewScorer  # noqa: E402
sc = synth.make_scene(5)
G = Gaussians(torch.from_numpy(sc.field.planes).cuda(), 3)
bv = int(sys.argv[1]) if len(sys.argv) > 1 else 64
s = ViewScorer(G, batch_views=bv, n_slots=2)
s.score_views(sc.cameras[:256])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s.score_views(sc.cameras)
e1.record()
torch.cuda.synchronize()
print("coarse pass ms", e0.elapsed_time(e1), "batch", bv)
