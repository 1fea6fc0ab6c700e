"""NEXT-3 refinement step on the GPU (gsr_l2_loss, gsr_adam_step through the
C ABI) vs oracle/optim.py, and a refinement run that recovers a perturbed
field from its own renders (UPDATE_GS, §4.1)."""
import numpy as np
import pytest
import torch

import synth
from oracle import optim
from tests.gpu_utils import to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


def test_l2_loss_and_gradient(ctx):
    from paper_2602_15355_b200 import gsr
    rng = np.random.default_rng(0)
    img, tgt = rng.random((3, 37, 23, 4)).astype(np.float32), rng.random((3, 37, 23, 4)).astype(np.float32)
    w = [1.0, 0.5, 2.0, 0.25]
    dl = torch.empty((3, 37, 23, 4), device="cuda")
    loss = gsr.gsr_l2_loss(ctx, torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), w, dl_dimg=dl)
    L, G = optim.l2_loss(img, tgt, w)
    assert abs(loss.item() - L) <= 1e-6 * L
    np.testing.assert_allclose(dl.cpu().numpy(), G, rtol=1e-5, atol=1e-9)


def test_adam_steps_vs_oracle(ctx):
    from paper_2602_15355_b200 import gsr
    rng = np.random.default_rng(1)
    P, n = 4, 1000
    p0 = rng.uniform(0.05, 0.95, (P, n, 4)).astype(np.float32)
    lr = rng.uniform(1e-3, 1e-2, (P, 4)).astype(np.float32)
    p, m, v = (torch.from_numpy(x).cuda() for x in (p0.copy(), np.zeros_like(p0), np.zeros_like(p0)))
    rp, rm, rv = p0.astype(np.float64), np.zeros_like(p0, np.float64), np.zeros_like(p0, np.float64)
    for t in range(1, 6):
        g = (rng.normal(size=(P, n, 4)) * 10.0 ** rng.uniform(-4, 0, (P, n, 4))).astype(np.float32)
        gsr.gsr_adam_step(ctx, p, torch.from_numpy(g).cuda(), m, v, lr, t)
        rp, rm, rv = optim.adam_step(rp, g, rm, rv, lr, t)
    torch.cuda.synchronize()
    np.testing.assert_allclose(p.cpu().numpy(), rp, rtol=2e-5, atol=1e-6)
    np.testing.assert_allclose(m.cpu().numpy(), rm, rtol=2e-5, atol=1e-8)  # float32 moments


def test_refinement_recovers_a_perturbed_field(ctx):
    """Captures = renders of the true field from 4 poses; the field with
    perturbed colours, opacities and positions is refined for 60 steps: the
    photometric loss drops by > 98 % (measured 0.0125 -> 6.4e-5)."""
    from paper_2602_15355_b200.pipeline import Refiner, Renderer
    fld, cams = synth.random_scene_small(3, 300, 64, 48, 55.0, 4, 0, logscale_mu=-2.4)
    true = to_dev(fld)
    targets = Renderer(true).forward(cams).clone()
    rng = np.random.default_rng(2)
    pert = fld.planes.copy()
    pert[3, :, :3] = np.clip(pert[3, :, :3] + rng.normal(0, 0.15, pert[3, :, :3].shape), 0, 1)
    pert[0, :, 3] = np.clip(pert[0, :, 3] * rng.uniform(0.6, 1.2, fld.n), 1e-3, 1.0)
    pert[0, :, :3] += rng.normal(0, 0.01, (fld.n, 3))
    G = to_dev(synth.GaussianField(pert.astype(np.float32), 0))
    lr = np.zeros((G.planes.shape[0], 4), np.float32)
    lr[0] = [1e-3, 1e-3, 1e-3, 2e-2]   # means, opacity
    lr[3] = [2e-2, 2e-2, 2e-2, 2e-2]   # DC colour
    ref = Refiner(G, lr)
    losses = [ref.step(cams, targets).item() for _ in range(60)]
    print("refinement loss", losses[0], "->", losses[-1])
    assert losses[-1] < 0.02 * losses[0], (losses[0], losses[-1])  # measured ~0.005
