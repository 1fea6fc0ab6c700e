"""Small driver for compute-sanitizer: every default
libgsr kernel on a configs[0]-shaped scene (2,000 Gaussians, 8 views 128^2,
SH 3 so every K1 path runs), plus the 64-bit depth-key fallback, the radix
tile sort, the NEXT-1..4 kernels and the u64 utility sort.  Exits 0 and
prints "sanitize_run ok" when every call returned GSR_OK.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import synth
    from paper_2602_15355_b200 import Context, Gaussians, gsr
    from paper_2602_15355_b200.pipeline import Refiner, Renderer, ViewScorer

    sc = synth.make_scene(2, n_override=2000, views=8)  # terrain generator, SH degree 3
    cams = synth.with_resolution(sc.cameras, 128, 128, 150.0)
    G = Gaussians(torch.from_numpy(sc.field.planes).cuda(), sc.field.sh_degree)
    # K1..K8: project, compact, depth onesweep, emit, ranges, K4c tile sort,
    # composite (variant 10) + part sums, score, select
    s = ViewScorer(G, batch_views=4, n_slots=2)
    scores = s.score_views(cams)
    s.select(scores, 3)
    # images, T_final, n_contrib, gray (NEXT-4 input) + Sobel
    ctx = Context(0)
    img = torch.empty((4, 128, 128, 4), device="cuda")
    sc4 = torch.empty(4, device="cuda")
    s.run_batch(cams[:4], sc4, images=img)
    r = Renderer(G)
    out = r.forward(cams[:2])
    r.backward(torch.ones_like(out))  # NEXT-3 K6b + K1b
    ref = Refiner(G, np.full((G.planes.shape[0], 4), 1e-4, np.float32))
    ref.step(cams[:2], out.clone())  # L2 loss + Adam
    gray = torch.rand((2, 128, 128), device="cuda")
    part = torch.empty(2 * 64, device="cuda")
    gsr.gsr_sobel_scores(ctx, gray, cams[:2], part, torch.empty(2, device="cuda"))
    mu = torch.rand((16, 5, 4, 256), device="cuda")
    gsr.gsr_w2_scores(ctx, mu, torch.rand_like(mu) + 0.1, torch.empty(16, device="cuda"))
    k = torch.randint(0, 2 ** 62, (5000,), dtype=torch.int64, device="cuda")
    v = torch.arange(5000, dtype=torch.int32, device="cuda")
    gsr.gsr_sort_pairs_u64(ctx, k, v, torch.empty_like(k), torch.empty_like(v))
    torch.cuda.synchronize()
    print("sanitize_run ok", scores.cpu().numpy()[:3], flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--variants":
        # the fallbacks in their own processes (libgsr reads GSR_* at context creation)
        for env in ({"GSR_DKEY64": "1"}, {"GSR_TSORT": "radix"}):
            r = subprocess.run([sys.executable, __file__], env=dict(os.environ, **env))
            if r.returncode:
                sys.exit(r.returncode)
    else:
        main()
