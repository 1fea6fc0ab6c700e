"""NEXT-4 parity: the Sobel image term of eq:uncert_img
through the C ABI -- K6's gray output and gsr_sobel_scores -- against
oracle/sobel.py (float64).  Gray images within 1e-6 absolute of the oracle's
channel mean of the oracle's composited RGB; scores within 1e-4 relative."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import sobel
from tests.gpu_utils import to_dev

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "sobel_examples.json")


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


def _cams(W, H):
    cams = np.zeros(1, dtype=synth.CAM_DTYPE)
    cams["width"], cams["height"] = W, H
    return cams


def _sobel_gpu(ctx, gray):
    from paper_2602_15355_b200 import gsr
    V, H, W = gray.shape
    cams = np.repeat(_cams(W, H), V)
    g = torch.from_numpy(np.ascontiguousarray(gray, dtype=np.float32)).cuda()
    part = torch.empty(V * ((W + 15) // 16) * ((H + 15) // 16), device="cuda")
    sc = torch.empty(V, device="cuda")
    gsr.gsr_sobel_scores(ctx, g, cams, part, sc)
    torch.cuda.synchronize()
    return sc.cpu().numpy().astype(np.float64)


def test_sobel_golden_through_abi(ctx):
    g = json.load(open(GOLDEN))
    for c in g["sobel"]:
        got = _sobel_gpu(ctx, np.array([c["gray"]], dtype=np.float32))[0]
        assert abs(got - c["expect"]) <= 1e-6 * max(1.0, c["expect"]), c["cite"]


@pytest.mark.parametrize("W,H,V", [(3, 3, 1), (37, 23, 3), (16, 16, 2), (130, 67, 4)])
def test_sobel_random_ragged(ctx, W, H, V):
    rng = np.random.default_rng(W * 1000 + H)
    gray = rng.random((V, H, W)).astype(np.float32)
    got = _sobel_gpu(ctx, gray)
    ref = np.array([sobel.sobel_magnitude(gray[v]).mean() for v in range(V)])
    np.testing.assert_allclose(got, ref, rtol=1e-5)


def test_sobel_rejects_small_images(ctx):
    from paper_2602_15355_b200 import gsr
    with pytest.raises(gsr.GsrError):
        _sobel_gpu(ctx, np.zeros((1, 2, 5), np.float32))


@pytest.mark.parametrize("cfg,views", [(1, 6), (2, 3)])
def test_scorer_image_term_vs_oracle(ctx, cfg, views):
    """ViewScorer with sobel_out: the mean-uncertainty scores (north_star) and
    the NEXT-4 image term of every view, vs the oracle's composite + Sobel."""
    from paper_2602_15355_b200.pipeline import ViewScorer
    sc = synth.make_scene(cfg, n_override=4000 if cfg == 1 else 20000, views=views)
    scorer = ViewScorer(to_dev(sc.field), batch_views=4)
    out = torch.empty(views, device="cuda")
    sob = torch.empty(views, device="cuda")
    scorer.score_views(sc.cameras, out, sobel_out=sob)
    torch.cuda.synchronize()
    ref_u, _, _, imgs = oracle.render_views(sc.field, sc.cameras, n_threads=4, images=True)
    np.testing.assert_allclose(out.cpu().numpy(), ref_u, rtol=1e-4)
    np.testing.assert_allclose(sob.cpu().numpy(), sobel.sobel_scores(imgs), rtol=1e-4)


def test_gray_output_matches_oracle_rgb(ctx):
    from tests.gpu_utils import gpu_batch, oracle_batch
    fld, cams = synth.random_scene_small(3, 300, 48, 40, 45.0, 2, 2, logscale_mu=-2.2)
    g = gpu_batch(ctx, fld, cams, images=True, want_unsorted=False, want_keys=False, want_gray=True)
    o = oracle_batch(fld, cams, images=True)
    ref = sobel.grayscale(o["rgbu"])
    assert np.abs(g["gray"].astype(np.float64) - ref).max() < 1e-6
