"""Pins of the NEXT-4 Sobel oracle (PAPER.md eq:uncert_img, L66-72; SPEC
sobel_gradient_scalar S:L239-248) against printed examples, closed forms and
scipy's own Sobel filter."""
import json
import os

import numpy as np
import pytest
from scipy import ndimage

from oracle import sobel

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sobel_examples.json")


def test_sobel_golden_examples():
    g = json.load(open(GOLDEN))
    for c in g["sobel"]:
        got = float(sobel.sobel_magnitude(np.array(c["gray"], dtype=np.float64)).mean())
        assert abs(got - c["expect"]) < 1e-12, c["cite"]


def test_sobel_linear_ramp_closed_form():
    """f = a x + b y on W x H: interior |grad| = 8 sqrt(a^2 + b^2) (central
    difference 2a times the 1-2-1 smoothing weight 4); a replicate-padded
    border column / row halves its own component."""
    W, H, a, b = 11, 7, 0.3, -0.2
    ys, xs = np.mgrid[0:H, 0:W]
    m = sobel.sobel_magnitude(a * xs + b * ys)
    fx = np.where((xs == 0) | (xs == W - 1), 4 * a, 8 * a)
    fy = np.where((ys == 0) | (ys == H - 1), 4 * b, 8 * b)
    np.testing.assert_allclose(m, np.sqrt(fx ** 2 + fy ** 2), rtol=1e-12, atol=1e-12)


def test_sobel_matches_scipy_nearest_mode():
    """Library pin: scipy.ndimage.sobel with mode='nearest' (= replicate
    padding) along each axis gives the same two components."""
    rng = np.random.default_rng(0)
    g = rng.random((13, 17))
    ref = np.hypot(ndimage.sobel(g, axis=1, mode="nearest"), ndimage.sobel(g, axis=0, mode="nearest"))
    np.testing.assert_allclose(sobel.sobel_magnitude(g), ref, rtol=1e-12, atol=1e-12)


def test_sobel_transpose_symmetry_and_grayscale():
    """Image vs its transpose -> equal scalars; grayscale is the
    channel mean, so equal channels reduce to the single-channel image."""
    rng = np.random.default_rng(1)
    rgb = rng.random((9, 12, 3))
    assert abs(sobel.sobel_score(rgb) - sobel.sobel_score(rgb.transpose(1, 0, 2))) < 1e-12
    c = rng.random((9, 12))
    assert abs(sobel.sobel_score(np.stack([c, c, c], -1)) - sobel.sobel_magnitude(c).mean()) < 1e-12
    with pytest.raises(ValueError):
        sobel.sobel_magnitude(np.zeros((2, 5)))
