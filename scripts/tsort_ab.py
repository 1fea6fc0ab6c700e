"""A/B of the tile sort (K4c counting scatter vs K4b radix) on configs[3]
(8,160 tiles per view) and the configs[4] fine pass (4,096 tiles per view)."""
import json
import os
import sys
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_15355_b200 import Gaussians  # noqa: E402
from paper_2602_15355_b200.pipeline import ViewScorer  # noqa: E402

def run(fld, cams, steps=3):
    G = Gaussians(torch.from_numpy(fld.planes).cuda(), fld.sh_degree)
    s = ViewScorer(G, batch_views=16, n_slots=2)
    for _ in range(2):
        s.score_views(cams)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        s.score_views(cams)
    e1.record()
    torch.cuda.synchronize()
    return round(len(cams) / (e0.elapsed_time(e1) / steps / 1e3), 1)

c4 = synth.make_scene(4)
c5 = synth.make_scene(5)
fine = synth.with_resolution(c5.cameras[:64], 1024, 1024, 1152.0)
print(json.dumps({"mode": os.environ.get("GSR_TSORT", "cs"), "c4": run(c4.field, c4.cameras),
                  "c5_fine": run(c5.field, fine)}))
