"""Pins of the NEXT-3 backward oracle (oracle/backward.py): its float64
forward reproduces the float32 oracle image; its autograd gradients match
central finite differences of that forward (frozen blend lists), and closed
forms for a single Gaussian."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import backward as bw
from tests.helpers import axis_camera, field_from


def _scene(seed=0, deg=1):
    fld, cams = synth.random_scene_small(seed, 60, 32, 24, 30.0, 1, deg, logscale_mu=-2.0)
    return fld, cams[0]


@pytest.mark.parametrize("deg", [0, 3])
def test_torch_forward_matches_float32_oracle(deg):
    fld, cam = _scene(1, deg)
    off, idx = bw.frozen_lists(fld, cam)
    img = bw.render_t(bw.params_from_field(fld), cam, deg, off, idx).detach().numpy()
    assert np.abs(img - oracle.render_view(fld, cam)["rgbu"]).max() < 2e-6


def test_torch_forward_matches_float32_oracle_with_alpha_clamp():
    """Opaque layers (o = 1) centred on pixel centres reach alpha = 0.99 (the
    O5 clamp) at those pixels: the float64 forward still reproduces the
    float32 oracle image there, and dL/do of a clamped pixel is zero (the
    clamp's derivative)."""
    cam = axis_camera(17, 17, 50.0, cx=8.5, cy=8.5)
    fld = field_from([[0, 0, 1.0], [0.02, -0.03, 1.6]], [[0.05] * 3] * 2, [[1, 0, 0, 0]] * 2, [1.0, 1.0],
                     [[1, 0.5, 0], [0, 0.5, 1]], [0.7, 0.2])
    off, idx = bw.frozen_lists(fld, cam)
    P = bw.params_from_field(fld)
    img = bw.render_t(P, cam, 0, off, idx)
    ref = oracle.render_view(fld, cam)["rgbu"]
    assert np.abs(img.detach().numpy() - ref).max() < 2e-6
    assert abs(float(ref[8, 8, 0]) - 0.99) < 1e-6  # the front layer's alpha is clamped at the centre
    # upstream gradient only at the clamped centre pixel: the front layer's
    # opacity gradient there is zero
    G = torch.zeros(17, 17, 4, dtype=torch.float64)
    G[8, 8] = 1.0
    (img * G).sum().backward()
    assert float(P["opac"].grad[0]) == 0.0


@pytest.mark.parametrize("deg", [1, 3])
def test_autograd_matches_central_differences(deg):
    """dL/dtheta (autograd) vs (L(theta + h) - L(theta - h)) / 2h of the same
    float64 forward with the blend lists frozen, for 60 random parameters of
    every kind (means, scales, raw quaternion, opacity, uncertainty, SH)."""
    fld, cam = _scene(2, deg)
    off, idx = bw.frozen_lists(fld, cam)
    rng = np.random.default_rng(3)
    G = torch.from_numpy(rng.normal(size=(int(cam["height"]), int(cam["width"]), 4)))
    P = bw.params_from_field(fld)
    (bw.render_t(P, cam, deg, off, idx) * G).sum().backward()
    used = np.unique(idx)
    checked = 0
    for name, t in P.items():
        for _ in range(10):
            g = int(rng.choice(used))
            j = tuple(int(rng.integers(0, s)) for s in t.shape[1:])
            h = 1e-6 * max(1.0, abs(float(t.data[(g,) + j])))
            vals = []
            for sgn in (1, -1):
                Q = {k: v.detach().clone() for k, v in P.items()}
                Q[name][(g,) + j] += sgn * h
                vals.append(float((bw.render_t(Q, cam, deg, off, idx) * G).sum()))
            fd = (vals[0] - vals[1]) / (2 * h)
            ad = float(t.grad[(g,) + j])
            assert abs(fd - ad) <= 1e-5 * max(1.0, abs(ad)), (name, g, j, fd, ad)
            checked += 1
    assert checked == 60


def test_single_gaussian_closed_forms():
    """One Gaussian (T = 1, alpha = o E < 0.99): C = o E (rgb, u), so
    dL/du = sum_p G_U o E, dL/do = sum_p E <G, (rgb, u)>, dL/drgb_ch = sum_p G_ch o E."""
    cam = axis_camera(40, 32, 60.0, cx=19.3, cy=15.8)
    o, rgb, unc = 0.6, [0.3, 0.5, 0.8], 0.4
    fld = field_from([[0.02, -0.01, 2.0]], [[0.12, 0.08, 0.1]], [[0.9, 0.1, -0.2, 0.3]], [o], [rgb], [unc])
    off, idx = bw.frozen_lists(fld, cam)
    P = bw.params_from_field(fld)
    rng = np.random.default_rng(0)
    G = rng.normal(size=(32, 40, 4))
    img = bw.render_t(P, cam, 0, off, idx)
    (img * torch.from_numpy(G)).sum().backward()
    o, rgb, unc = float(np.float32(o)), [float(np.float32(c)) for c in rgb], float(np.float32(unc))
    u, v, A, B, C, oo, col = bw.project_t({k: t.detach() for k, t in P.items()}, cam, 0)
    ys, xs = np.mgrid[0:32, 0:40]
    dx, dy = float(u[0]) - (xs + 0.5), float(v[0]) - (ys + 0.5)
    E = np.exp(-0.5 * (float(A[0]) * dx * dx + float(C[0]) * dy * dy) - float(B[0]) * dx * dy)
    on = (np.diff(off) > 0).reshape(32, 40)
    Ek = np.where(on, E, 0.0)
    np.testing.assert_allclose(float(P["unc"].grad[0]), (G[..., 3] * o * Ek).sum(), rtol=1e-10)
    np.testing.assert_allclose(float(P["opac"].grad[0]), (Ek * (G[..., :3] @ np.array(rgb) + G[..., 3] * unc)).sum(),
                               rtol=1e-10)
    np.testing.assert_allclose(P["sh"].grad[0, 0].numpy(), [(G[..., c] * o * Ek).sum() for c in range(3)], rtol=1e-10)
