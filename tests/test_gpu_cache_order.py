"""NEXT-2b parity: cached view-direction orderings on the GPU
(gsr_build_order_cache + gsr_bin_sort_cached, through the C ABI) vs
oracle/cache_order.py: bit-exact orderings, sorted values and ranges, images
within 1e-4 (expected bit-exact), scores within 1e-4 relative."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import cache_order as co
from tests.gpu_utils import to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


def _tiles_small(fld, k=3):
    start = np.linspace(0, fld.n, k + 1).round().astype(np.int64)
    centres = np.array([fld.planes[0, start[t]:start[t + 1], :3].mean(0) for t in range(k)], dtype=np.float64)
    return start, centres


def test_cache_orderings_bit_exact(ctx):
    from paper_2602_15355_b200 import gsr
    fld, _ = synth.random_scene_small(1, 700, 48, 40, 45.0, 1, 1)
    start, centres = _tiles_small(fld)
    bins = np.array([8, 16, 8], np.int32)
    oc = gsr.OrderCache(ctx, to_dev(fld), start, bins, centres)
    torch.cuda.synchronize()
    got = oc.cache.cpu().numpy().view(np.uint32)
    ref = np.concatenate([co.cached_orders(fld, start, int(bins[t]), t).reshape(-1) for t in range(3)])
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("seed,deg,W,H", [(0, 0, 48, 40), (2, 3, 100, 37), (3, 1, 16, 16)])
def test_cached_batch_vs_oracle(ctx, seed, deg, W, H):
    from paper_2602_15355_b200 import gsr
    fld, cams = synth.random_scene_small(seed, 700, W, H, 0.9 * max(W, H), 3, deg, logscale_mu=-2.6)
    start, centres = _tiles_small(fld)
    bins = np.array([8, 8, 16], np.int32)
    G = to_dev(fld)
    oc = gsr.OrderCache(ctx, G, start, bins, centres)
    V, n = len(cams), fld.n
    T = V * ((W + 15) // 16) * ((H + 15) // 16)
    rec = torch.zeros((V, n, 12), device="cuda")
    binr = torch.zeros(10 * V * n, dtype=torch.int32, device="cuda")
    gsr.gsr_project(ctx, G, cams, rec, binr)
    ranges = torch.zeros((T, 2), dtype=torch.int32, device="cuda")
    vals = torch.zeros(4 * n * V + 16, dtype=torch.int32, device="cuda")
    K = gsr.gsr_bin_sort_cached(ctx, binr, n, cams, oc, vals, vals.numel(), ranges)
    part = torch.zeros(T, device="cuda")
    rgbu = torch.zeros((V, H, W, 4), device="cuda")
    gsr.gsr_composite(ctx, rec, n, vals, ranges, cams, part, rgbu=rgbu)
    torch.cuda.synchronize()
    tpv = T // V
    gv = vals.cpu().numpy().view(np.uint32)[:K]
    gr = ranges.cpu().numpy().view(np.uint32)
    base = 0
    for v, cam in enumerate(cams):
        o = co.render_view_cached(fld, cam, start, bins, centres)
        kv = len(o["vals"])
        assert np.array_equal(gv[base:base + kv], o["vals"]), f"view {v} vals"
        assert np.array_equal(gr[v * tpv:(v + 1) * tpv] - base, o["ranges"]), f"view {v} ranges"
        assert np.array_equal(rgbu[v].cpu().numpy(), o["rgbu"]), f"view {v} image"
        base += kv
    assert base == K


def test_flyover_scorer_cached_vs_oracle(ctx):
    """configs[3] geometry (4,000 Gaussians per tile), fly-over views at
    480x270: ViewScorer with the order cache vs the oracle's cached render."""
    from paper_2602_15355_b200.pipeline import ViewScorer
    fld = synth.gen_config4_field(4_000)
    start, centres = synth.config4_tiles(4_000)
    bins = [co.bins_for(u) for u in co.tile_mean_uncertainty(fld, start)]
    cams = synth.with_resolution(synth.flyover_cameras(64, 1920, 1080, 1500.0)[::8], 480, 270, 375.0)
    sc = ViewScorer(to_dev(fld), batch_views=4, order_tiles=(start, bins, centres))
    got = sc.score_views(cams).cpu().numpy()
    ref = np.array([co.render_view_cached(fld, c, start, bins, centres)["score"] for c in cams])
    np.testing.assert_allclose(got, ref, rtol=1e-4)


def test_cache_policy_bins_in_libgsr(ctx):
    """gsr_order_cache_bins (pipeline.cache_bins) = the oracle's policy
    (§3.5, tau = 0.6): per tile, 16 bins if its mean
    uncertainty exceeds tau, else 8 -- on the configs[3] tiles, on tiles made
    hot / cold on purpose, and for a tau just below / above one tile's mean."""
    from paper_2602_15355_b200 import gsr
    from paper_2602_15355_b200.pipeline import cache_bins
    fld = synth.gen_config4_field(4_000)
    start, _ = synth.config4_tiles(4_000)
    planes = fld.planes.copy()
    planes[1, start[1]:start[2], 3] = 0.9  # hot tile
    planes[1, start[2]:start[3], 3] = 0.1  # cold tile
    fld = synth.GaussianField(planes, fld.sh_degree)
    G = to_dev(fld)
    means = co.tile_mean_uncertainty(fld, start)
    want = np.array([co.bins_for(u) for u in means], np.int32)
    got = cache_bins(G, start, ctx=ctx)
    assert np.array_equal(got, want) and got[1] == 16 and got[2] == 8
    for tau, hot in ((means[0] * (1 - 1e-6), 16), (means[0] * (1 + 1e-6), 8)):
        b = gsr.gsr_order_cache_bins(ctx, G, start, float(tau))
        assert b[0] == hot and np.array_equal(b, [co.bins_for(u, float(np.float32(tau))) for u in means])
    with pytest.raises(gsr.GsrError):
        gsr.gsr_order_cache_bins(ctx, G, np.asarray(start)[:-1], 0.6)  # does not cover [0, n)
