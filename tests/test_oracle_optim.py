"""Pins of the NEXT-3 refinement-step oracle: Adam against torch.optim.Adam
(library routine), the L2 loss gradient against central finite differences,
and the projection onto the parameters' domain."""
import numpy as np
import torch

from oracle import optim


def test_adam_matches_torch_optim_adam():
    rng = np.random.default_rng(0)
    P, n = 4, 50
    p0 = rng.uniform(0.1, 0.9, (P, n, 4))
    lr = rng.uniform(1e-3, 1e-2, (P, 4))
    p, m, v = p0.copy(), np.zeros_like(p0), np.zeros_like(p0)
    tp = [torch.tensor(p0[i, :, c].copy(), requires_grad=True) for i in range(P) for c in range(4)]
    opt = torch.optim.Adam([{"params": [tp[i * 4 + c]], "lr": float(lr[i, c])} for i in range(P) for c in range(4)],
                           betas=(0.9, 0.999), eps=1e-8)
    for t in range(1, 6):
        g = rng.normal(size=(P, n, 4)) * 1e-3  # small steps stay inside the projection's box
        p, m, v = optim.adam_step(p, g, m, v, lr, t)
        for i in range(P):
            for c in range(4):
                tp[i * 4 + c].grad = torch.tensor(g[i, :, c].copy())
        opt.step()
        ref = np.stack([np.stack([tp[i * 4 + c].detach().numpy() for c in range(4)], -1) for i in range(P)])
        np.testing.assert_allclose(p, ref, rtol=1e-12, atol=1e-14)


def test_adam_projection():
    p = np.zeros((3, 2, 4)) + 0.5
    g = np.zeros_like(p)
    g[0, :, 3] = [-1.0, 1.0]    # push opacity up / down
    g[1, :, 0] = 1.0            # push a scale below 0
    g[1, :, 3] = 1.0            # push uncertainty below 0
    lr = np.full((3, 4), 10.0)
    q, _, _ = optim.adam_step(p, g, np.zeros_like(p), np.zeros_like(p), lr, 1)
    assert q[0, 0, 3] == 1.0 and q[0, 1, 3] == 1e-4
    assert np.all(q[1, :, 0] == 1e-6) and np.all(q[1, :, 3] == 0.0)


def test_l2_loss_gradient_by_central_differences():
    rng = np.random.default_rng(1)
    img, tgt = rng.random((2, 5, 6, 4)), rng.random((2, 5, 6, 4))
    w = [1.0, 0.5, 2.0, 0.25]
    L, G = optim.l2_loss(img, tgt, w)
    assert abs(L - (np.array(w) * (img - tgt) ** 2).sum() / 60) < 1e-14
    h = 1e-6
    for idx in [(0, 0, 0, 0), (1, 4, 5, 3), (0, 2, 3, 1)]:
        a, b = img.copy(), img.copy()
        a[idx] += h
        b[idx] -= h
        fd = (optim.l2_loss(a, tgt, w)[0] - optim.l2_loss(b, tgt, w)[0]) / (2 * h)
        assert abs(fd - G[idx]) < 1e-8
