"""NEXT-3 parity: the backward rasterizer (gsr_backward: K6b + K1b, through
the C ABI) vs oracle/backward.py (float64 autograd over the float32 forward's
blend lists).  Bar: for every parameter kind (means, opacity, scales,
uncertainty, quaternion, SH), max |gpu - oracle| <= 5e-5 x max |oracle| of
that kind (float32 chain rule + float atomics vs float64; measured <= 4e-6)."""
import numpy as np
import pytest

import synth
from oracle import backward as bw
from tests.gpu_utils import gpu_forward_backward

pytestmark = pytest.mark.gpu

KINDS = {"means": (0, slice(0, 3)), "opacity": (0, slice(3, 4)), "scales": (1, slice(0, 3)),
         "uncertainty": (1, slice(3, 4)), "quaternion": (2, slice(0, 4))}


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


def _compare(got, ref, deg, rtol=5e-5):
    worst = {}
    for name, (pl, sl) in list(KINDS.items()) + [("sh", (slice(3, None), slice(None)))]:
        g, r = got[pl][..., sl], ref[pl][..., sl]
        scale = np.abs(r).max()
        err = np.abs(g - r).max()
        worst[name] = (err, scale)
        assert err <= rtol * scale + 1e-7, (name, err, scale)
    return worst


@pytest.mark.parametrize("seed,deg,W,H,views", [(0, 0, 48, 40, 1), (1, 1, 33, 17, 2), (2, 3, 64, 48, 2),
                                                (3, 2, 40, 40, 3)])
def test_backward_small_scenes(ctx, seed, deg, W, H, views):
    fld, cams = synth.random_scene_small(seed, 150, W, H, 0.9 * max(W, H), views, deg, logscale_mu=-2.4)
    G = np.random.default_rng(seed).normal(size=(views, H, W, 4)).astype(np.float32)
    img, got = gpu_forward_backward(ctx, fld, cams, G)
    ref = bw.backward_views(fld, cams, G)
    w = _compare(got, ref, deg)
    print({k: f"{e:.2e}/{s:.2e}" for k, (e, s) in w.items()})


def test_backward_with_lod(ctx):
    fld, cams = synth.random_scene_small(4, 150, 48, 40, 45.0, 2, 1, logscale_mu=-2.4)
    lod = synth.random_lod(np.random.default_rng(4), fld.n)
    G = np.random.default_rng(5).normal(size=(2, 40, 48, 4)).astype(np.float32)
    img, got = gpu_forward_backward(ctx, fld, cams, G, lod=lod)
    ref = bw.backward_views(fld, cams, G, lod=lod)
    _compare(got, ref, 1)


def test_backward_is_linear_and_zero_for_zero_upstream(ctx):
    fld, cams = synth.random_scene_small(6, 120, 32, 32, 30.0, 1, 1, logscale_mu=-2.4)
    G = np.random.default_rng(6).normal(size=(1, 32, 32, 4)).astype(np.float32)
    _, g1 = gpu_forward_backward(ctx, fld, cams, G)
    _, g2 = gpu_forward_backward(ctx, fld, cams, 2 * G)
    _, g0 = gpu_forward_backward(ctx, fld, cams, 0 * G)
    assert not g0.any()
    np.testing.assert_allclose(g2, 2 * g1, rtol=1e-4, atol=1e-6 * np.abs(g1).max())


def test_renderer_api_matches_oracle(ctx):
    """pipeline.Renderer (the UPDATE_GS building block): forward image equals
    the oracle's; backward gradients match the float64 autograd oracle."""
    import torch
    import oracle
    from paper_2602_15355_b200.pipeline import Renderer
    from tests.gpu_utils import to_dev
    fld, cams = synth.random_scene_small(7, 200, 48, 40, 45.0, 2, 3, logscale_mu=-2.4)
    r = Renderer(to_dev(fld))
    img = r.forward(cams)
    ref_img = np.stack([oracle.render_view(fld, c)["rgbu"] for c in cams])
    assert np.array_equal(img.cpu().numpy(), ref_img)
    G = np.random.default_rng(8).normal(size=ref_img.shape).astype(np.float32)
    got = r.backward(torch.from_numpy(G).cuda()).cpu().numpy()
    _compare(got, bw.backward_views(fld, cams, G), 3)


@pytest.mark.parametrize("red", ["0", "2", "2 GSR_BWNW=8"])
def test_backward_reduction_variants(ctx, red, monkeypatch):
    """K6b's warp reductions (shuffle trees / transposed butterfly, GSR_BWRED)
    and block shapes (2-warp sub-tile blocks / one 8-warp block per tile,
    GSR_BWNW) give the same gradients within the float tolerance."""
    from paper_2602_15355_b200 import Context
    red, *extra = red.split()
    monkeypatch.setenv("GSR_BWRED", red)
    for kv in extra:
        k, v = kv.split("=")
        monkeypatch.setenv(k, v)
    c = Context(0)
    fld, cams = synth.random_scene_small(8, 150, 40, 33, 40.0, 2, 2, logscale_mu=-2.4)
    G = np.random.default_rng(9).normal(size=(2, 33, 40, 4)).astype(np.float32)
    img, got = gpu_forward_backward(c, fld, cams, G)
    _compare(got, bw.backward_views(fld, cams, G), 2)


def test_backward_alpha_clamp(ctx):
    """Opaque layers (o = 1) reach the alpha = 0.99 clamp at their centres,
    where K6b's power and opacity gradients must vanish: gradients match the
    float64 oracle on a scene of such layers."""
    from tests.helpers import axis_camera, field_from
    rng = np.random.default_rng(11)
    n = 12
    means = np.stack([rng.uniform(-0.2, 0.2, n), rng.uniform(-0.2, 0.2, n), 1.0 + 0.2 * np.arange(n)], 1)
    means[::3, :2] = 0.0  # every third layer on the axis: its mean projects onto the centre of pixel (16, 14)
    fld = field_from(means, [[0.06] * 3] * n, [[1, 0, 0, 0]] * n, [1.0] * n, rng.uniform(0, 1, (n, 3)),
                     rng.uniform(0, 1, n))
    # cx, cy on a pixel centre: o exp(0) = 1 > 0.99 there, so alpha is clamped
    cams = np.stack([axis_camera(33, 29, 60.0, cx=16.5, cy=14.5)])
    G = rng.normal(size=(1, 29, 33, 4)).astype(np.float32)
    img, got = gpu_forward_backward(ctx, fld, cams, G)
    _compare(got, bw.backward_views(fld, cams, G), 0)
