"""NEXT-3 oracle: the refinement step of UPDATE_GS ("bounded refinement",
PAPER.md §4.1) -- TEST INFRASTRUCTURE ONLY (same rules as the package
docstring of oracle/).

  l2_loss     L = (1/N) sum_p sum_ch w_ch (C - T)^2, dL/dC = (2/N) w (C - T)
  adam_step   Adam, Kingma & Ba 2015 Algorithm 1 (bias-corrected moments),
              written out per component in float64, then the projection the
              DESIGN.md reading fixes: opacity in [1e-4, 1], scales >= 1e-6,
              uncertainty >= 0.
Pins: tests/test_oracle_optim.py (torch.optim.Adam, finite differences).
"""
from __future__ import annotations

import numpy as np


def l2_loss(img, target, weights):
    img = np.asarray(img, dtype=np.float64)
    t = np.asarray(target, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64).reshape(4)
    d = img - t
    n = d.size // 4
    return float((w * d * d).sum() / n), 2.0 * w * d / n


def adam_step(p, g, m, v, lr, t, beta1=0.9, beta2=0.999, eps=1e-8):
    """One Adam step on plane-layout arrays [P][n][4]; lr [P][4]; returns (p, m, v)."""
    p = np.asarray(p, dtype=np.float64).copy()
    g = np.asarray(g, dtype=np.float64)
    m = beta1 * np.asarray(m, dtype=np.float64) + (1 - beta1) * g
    v = beta2 * np.asarray(v, dtype=np.float64) + (1 - beta2) * g * g
    mh = m / (1 - beta1 ** t)
    vh = v / (1 - beta2 ** t)
    p = p - np.asarray(lr, dtype=np.float64)[:, None, :] * mh / (np.sqrt(vh) + eps)
    p[0, :, 3] = np.clip(p[0, :, 3], 1e-4, 1.0)
    p[1, :, :3] = np.maximum(p[1, :, :3], 1e-6)
    p[1, :, 3] = np.maximum(p[1, :, 3], 0.0)
    return p, m, v
