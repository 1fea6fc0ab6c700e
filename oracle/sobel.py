"""NEXT-4 oracle: the image-space spatial-frequency term of PAPER.md
eq:uncert_img (§3.3) -- TEST INFRASTRUCTURE ONLY (same rules as the
package docstring of oracle/).

    u_img(theta) = || grad I(theta) ||_2  (+ lambda LPIPS, out of scope)

"grad is computed using a 3x3 Sobel operator and the result is reduced to a
scalar via per-pixel Euclidean norm and global average" (L72).  Readings
(DESIGN.md): the image is the rendered RGB of the view (the north_star
renders instead of sampling the diffusion mean); grayscale = mean of the
three channels, Sobel-x / Sobel-y with replicate padding (S:L241-244
sobel_gradient_scalar); per-pixel sqrt(gx^2 + gy^2); mean over all W*H
pixels.  Plain float64 loops over the 3x3 taps, in the definition's order.
Pins: tests/test_oracle_sobel.py.
"""
from __future__ import annotations

import numpy as np

# Sobel-x taps K[dy+1][dx+1]; Sobel-y is its transpose.
SOBEL_X = ((-1.0, 0.0, 1.0), (-2.0, 0.0, 2.0), (-1.0, 0.0, 1.0))


def grayscale(rgb):
    """Mean of the three channels, float64 [H][W] (rgb: [H][W][>=3])."""
    a = np.asarray(rgb, dtype=np.float64)
    return (a[..., 0] + a[..., 1] + a[..., 2]) / 3.0


def sobel_magnitude(gray):
    """Per-pixel Euclidean norm of (Sobel-x, Sobel-y), replicate padding."""
    g = np.asarray(gray, dtype=np.float64)
    H, W = g.shape
    if H < 3 or W < 3:
        raise ValueError("image smaller than the 3x3 kernel (S:L243)")
    gx = np.zeros((H, W))
    gy = np.zeros((H, W))
    for dy in (-1, 0, 1):
        rows = np.clip(np.arange(H) + dy, 0, H - 1)
        for dx in (-1, 0, 1):
            cols = np.clip(np.arange(W) + dx, 0, W - 1)
            v = g[rows][:, cols]
            gx += SOBEL_X[dy + 1][dx + 1] * v
            gy += SOBEL_X[dx + 1][dy + 1] * v
    return np.sqrt(gx * gx + gy * gy)


def sobel_score(rgb):
    """u_img without the LPIPS term: global mean of the gradient magnitude."""
    return float(sobel_magnitude(grayscale(rgb)).mean())


def sobel_scores(images):
    """Per-view scores for [V][H][W][>=3] images."""
    return np.array([sobel_score(im) for im in images], dtype=np.float64)
