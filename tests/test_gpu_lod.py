"""NEXT-2 parity: LOD blending in K1 (PAPER.md eq:lod_blend, clamped form of
App. A.4) through the C ABI vs the oracle -- the same bar as the base path:
bit-exact bin records, keys, order and ranges; images within 1e-4 (expected
bit-exact); scores within 1e-4 relative."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gpu_utils import to_dev, to_dev_lod
from tests.test_gpu_parity import _full_check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


@pytest.mark.parametrize("seed,deg,W,H", [(0, 0, 48, 40), (1, 3, 100, 37), (2, 1, 16, 16)])
def test_lod_small_scenes(ctx, seed, deg, W, H):
    fld, cams = synth.random_scene_small(seed, 700, W, H, 0.9 * max(W, H), 3, deg, logscale_mu=-2.6)
    lod = synth.random_lod(np.random.default_rng(seed), fld.n)
    g, o = _full_check(ctx, fld, cams, lod=lod)
    assert np.array_equal(g["rgbu"], o["rgbu"])
    # the weights really vary: some pairs culled by LOD, others scaled
    base = [oracle.project(fld, c) for c in cams]
    assert sum(int(((b["n_tiles"] > 0) & (p["n_tiles"] == 0)).sum()) for b, p in zip(base, o["projs"])) > 0


def test_lod_wang_tiles_flyover(ctx):
    """Config-4 geometry with six LOD levels per Wang tile (reduced draws), 4
    fly-over views at 1920x1080: LOD-blended scores through ViewScorer vs the
    oracle, and the LOD render differs from the level-0-only render."""
    from paper_2602_15355_b200.pipeline import ViewScorer
    fld, lod = synth.gen_config4_lod(n_per_tile=2048)
    cams = synth.flyover_cameras(64, 1920, 1080, 1500.0)[::16]
    scorer = ViewScorer(to_dev(fld), batch_views=4, lod=to_dev_lod(lod))
    got = scorer.score_views(cams).cpu().numpy()
    ref, _, _, _ = oracle.render_views(fld, cams, n_threads=4, lod=lod)
    np.testing.assert_allclose(got, ref, rtol=1e-4)
    full, _, _, _ = oracle.render_views(fld, cams, n_threads=4)
    assert np.abs(full - ref).max() > 1e-3
