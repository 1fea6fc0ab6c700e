"""Adversarial parity cases for K6's culls.

K6 skips a list entry for a warp's 8x4 pixel box when (a) the box misses the
fp16 round-up AABB of the entry's alpha >= 1/255 ellipse, or (b) the conic's
minimum over the box (an edge minimum, rcp.approx for the minimiser) exceeds
the skip bound with slack.  Both are exact only if they never skip an entry
that blends somewhere in the box; these scenes push each to its limits, and
the images, T_final and n_contrib must stay bit-identical to the oracle
(which has no culls), whose tiled result is itself checked against its
brute-force composite.

  huge_offscreen   sigma' ~ 4e4 px, mean ~ 7e4 px off-screen: the extents
                   exceed the fp16 range (65,504)
  needles          eigenvalue ratios 1e6 .. 1e9, any in-plane angle, means up
                   to ~2,000 px from the boxes they cross (edge minima by
                   cancellation: A dx^2 ~ 2 B dx dy ~ C dy^2)
  near_plane       depths just above znear far outside the 1.3x FOV clamp
  corner_grazers   small ellipses whose alpha >= 1/255 boundary grazes warp-box
                   corners and edges (means just outside the boxes)
"""
import numpy as np
import pytest

import oracle
from tests.gpu_utils import gpu_batch, oracle_batch
from tests.helpers import axis_camera, field_from, random_unit_quats

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


def _rot_z(angle):
    """Unit quaternion (w, x, y, z) of a rotation by `angle` about +z."""
    return [np.cos(angle / 2), 0.0, 0.0, np.sin(angle / 2)]


def _field_huge_offscreen(rng):
    # camera at the origin looking down +z, f = 64, 64 x 64 (cx = 32):
    # xn = x / z ~ 1100 >> limx = 0.65, so the mean projects ~70,000 px right of
    # the image while the clamped Jacobian keeps sigma'_x ~ 4e4 px
    n = 6
    means = np.stack([rng.uniform(1800, 2600, n) * rng.choice([-1, 1], n), rng.uniform(-300, 300, n),
                      np.full(n, 2.0)], 1)
    scales = np.full((n, 3), 1000.0)
    bg = 12  # ordinary Gaussians in front of and behind them
    mb = np.stack([rng.uniform(-0.4, 0.4, bg), rng.uniform(-0.4, 0.4, bg), rng.uniform(1.0, 3.0, bg)], 1)
    sb = np.exp(rng.normal(-3.0, 0.4, (bg, 3)))
    return field_from(np.concatenate([means, mb]), np.concatenate([scales, sb]), random_unit_quats(rng, n + bg),
                      rng.uniform(0.3, 0.9, n + bg), rng.uniform(0, 1, (n + bg, 3)), rng.uniform(0, 1, n + bg))


def _field_needles(rng):
    n = 40
    ang = rng.uniform(0, np.pi, n)
    q = np.array([_rot_z(a) for a in ang])
    tilt = random_unit_quats(rng, n) * 0.02 + np.array([1.0, 0, 0, 0])  # slight out-of-plane tilt
    tilt /= np.linalg.norm(tilt, axis=1, keepdims=True)
    # compose: q * tilt (Hamilton product)
    w1, x1, y1, z1 = q.T
    w2, x2, y2, z2 = tilt.T
    qq = np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                   w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], 1)
    z = rng.uniform(1.5, 3.0, n)
    # major axis along local x (the in-plane angle turns it), 1e-5 .. 1e-6 minor axes
    scales = np.stack([rng.uniform(30.0, 150.0, n), 10 ** rng.uniform(-6, -4.5, n), 10 ** rng.uniform(-6, -4.5, n)], 1)
    # the mean slides along the needle up to ~2,000 px away from the image
    off = rng.uniform(-2000.0, 2000.0, n) * z / 64.0
    means = np.stack([off * np.cos(ang) + rng.uniform(-0.2, 0.2, n) * z / 2,
                      off * np.sin(ang) + rng.uniform(-0.2, 0.2, n) * z / 2, z], 1)
    return field_from(means, scales, qq, rng.uniform(0.2, 1.0, n), rng.uniform(0, 1, (n, 3)), rng.uniform(0, 1, n))


def _field_near_plane(rng):
    n = 80
    z = rng.uniform(0.2001, 0.26, n)
    xn = rng.uniform(-3.0, 3.0, n)
    yn = rng.uniform(-3.0, 3.0, n)
    means = np.stack([xn * z, yn * z, z], 1)
    scales = np.exp(rng.normal(-3.5, 0.8, (n, 3)))
    return field_from(means, scales, random_unit_quats(rng, n), rng.uniform(0.1, 1.0, n), rng.uniform(0, 1, (n, 3)),
                      rng.uniform(0, 1, n))


def _field_corner_grazers(rng):
    # warp boxes are 8 x 4 px at multiples of (8, 4): put small isotropic
    # Gaussians at a box corner or edge midpoint, pushed out by ~its alpha
    # boundary radius so the boundary grazes the box
    n = 400
    f, z = 64.0, 2.0
    sig_px = rng.uniform(0.6, 3.0, n)
    o = rng.uniform(0.05, 1.0, n)
    r = np.sqrt(np.maximum(2.0 * np.log(255.0 * o), 0.0)) * np.sqrt(sig_px ** 2 + 0.3)
    bx = rng.integers(0, 8, n) * 8.0
    by = rng.integers(0, 16, n) * 4.0
    kind = rng.integers(0, 3, n)
    ang = rng.uniform(0, 2 * np.pi, n)
    px = np.where(kind == 0, bx, np.where(kind == 1, bx + 4.0, bx)) + 0.5
    py = np.where(kind == 0, by, np.where(kind == 1, by, by + 2.0)) + 0.5
    px = px + (r + rng.uniform(-0.05, 0.05, n)) * np.cos(ang)
    py = py + (r + rng.uniform(-0.05, 0.05, n)) * np.sin(ang)
    means = np.stack([(px - 32.0) * z / f, (py - 32.0) * z / f, np.full(n, z) + rng.uniform(0, 0.5, n)], 1)
    s = sig_px * z / f
    return field_from(means, np.stack([s, s, s], 1), random_unit_quats(rng, n), o, rng.uniform(0, 1, (n, 3)),
                      rng.uniform(0, 1, n))


CASES = {"huge_offscreen": _field_huge_offscreen, "needles": _field_needles, "near_plane": _field_near_plane,
         "corner_grazers": _field_corner_grazers}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("seed", [0, 1])
def test_culls_stay_exact(ctx, case, seed):
    rng = np.random.default_rng(100 + seed)
    fld = CASES[case](rng)
    cams = np.stack([axis_camera(64, 64, 64.0)] * 2)
    g = gpu_batch(ctx, fld, cams, want_unsorted=False)
    o = oracle_batch(fld, cams)
    assert g["K"] == len(o["vals"]) and np.array_equal(g["vals"], o["vals"]), case
    for v in range(len(cams)):
        bf = oracle.composite_brute(o["projs"][v], cams[v])
        assert np.array_equal(bf["rgbu"], o["rgbu"][v]), case  # the reference itself: tiled == brute force
    assert np.array_equal(g["n_contrib"], o["n_contrib"]), (case, int((g["n_contrib"] != o["n_contrib"]).sum()))
    assert np.array_equal(g["t_final"], o["t_final"]), case
    assert np.array_equal(g["rgbu"], o["rgbu"]), (case, np.abs(g["rgbu"] - o["rgbu"]).max())
    assert g["n_frag"] == o["n_frag"] and g["n_eval"] == o["n_eval"]
    # the case must actually exercise what it targets
    vis = o["projs"][0]["n_tiles"] > 0
    assert vis.sum() > 0 and o["n_frag"] > 0, case
