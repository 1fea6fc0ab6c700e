"""NEXT-3 profiling driver: forward + backward of one 16-view c3 batch, three
times (for ncu launch lists and full-set captures of K6b / K1b).
    python scripts/backward_once.py"""
import sys, torch
sys.path.insert(0, ".")
import synth
from paper_2602_15355_b200 import Gaussians
from paper_2602_15355_b200.pipeline import Renderer
sc = synth.make_scene(3)
G = Gaussians(torch.from_numpy(sc.field.planes).cuda(), 3)
cams = synth.fibonacci_cameras(1024, 4.0, 800, 800, 900.0)[::64]
r = Renderer(G)
img = r.forward(cams)
target = img + 0.01 * torch.randn_like(img)
grads = torch.zeros_like(G.planes)
for _ in range(3):
    img = r.forward(cams)
    r.backward(2.0 * (img - target), grads)
torch.cuda.synchronize()
print("ok")
