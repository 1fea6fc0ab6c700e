"""Time one forward + backward of a 16-view c3 batch (device events)."""
import sys
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2602_15355_b200 import Gaussians  # noqa: E402
from paper_2602_15355_b200.pipeline import Renderer  # noqa: E402
sc = synth.make_scene(3, views=16)
G = Gaussians(torch.from_numpy(sc.field.planes).cuda(), 3)
r = Renderer(G)
g = torch.randn((16, 800, 800, 4), device="cuda")
grads = torch.zeros_like(G.planes)
for _ in range(2):
    r.forward(sc.cameras)
    r.backward(g, grads)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
r.forward(sc.cameras)
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    r.backward(g, grads)
e1.record()
torch.cuda.synchronize()
print("backward ms", e0.elapsed_time(e1) / 5)
