import sys, torch, numpy as np
sys.path.insert(0, '.')
import synth
from paper_2602_15355_b200 import Gaussians
from paper_2602_15355_b200.pipeline import Renderer
sc = synth.make_scene(3, views=16)
G = Gaussians(torch.from_numpy(sc.field.planes).cuda(), 3)
r = Renderer(G)
img = r.forward(sc.cameras)
g = torch.randn_like(img)
grads = torch.zeros_like(G.planes)
for _ in range(3):
    img = r.forward(sc.cameras)
    r.backward(g, grads)
torch.cuda.synchronize()
print("ok")
