"""Pins of the NEXT-2b cached-ordering oracle (§3.5;
SPEC lod-cache S:L571-591): valid sorted permutations, the tau policy,
exactness when the view looks along a bin direction, and the fidelity bound
of cached vs exact ordering on the fly-over scene."""
import math

import numpy as np

import oracle
import synth
from oracle import cache_order as co
from tests.helpers import field_from


def test_orderings_are_sorted_permutations():
    """every cached ordering is a permutation of the tile and sorted by
    the bin's key (Python's comparison sort on (key, index) as the oracle)."""
    fld, _ = synth.random_scene_small(0, 300, 48, 40, 45.0, 1, 0)
    start = np.array([0, 120, 300])
    for t in range(2):
        for B in (8, 16):
            C = co.cached_orders(fld, start, B, t)
            dirs = co.bin_dirs(B)
            for k in range(B):
                idx = list(range(start[t], start[t + 1]))
                x = fld.planes[0, :, 0].astype(np.float32)
                z = fld.planes[0, :, 2].astype(np.float32)
                key = lambda g: (float(np.float32(x[g] * dirs[k, 0]) + np.float32(z[g] * dirs[k, 1])), g)  # noqa: E731
                assert C[k].tolist() == sorted(idx, key=key)


def test_cache_policy():
    """S:L576-577 (u_bar 0.9 -> 16 bins, 0.1 -> 8 at tau = 0.6) and S:L593
    (raising tau never increases a tile's bin count)."""
    assert co.bins_for(0.9) == 16 and co.bins_for(0.1) == 8 and co.bins_for(0.6) == 8
    for u in np.linspace(0, 1, 21):
        assert all(co.bins_for(u, t2) <= co.bins_for(u, t1) for t1, t2 in [(0.2, 0.4), (0.4, 0.8)])


def test_cached_equals_exact_when_looking_along_a_bin():
    """Camera looking horizontally along +x = bin 0: the cached order is the
    depth order, so the render equals the exact-sort render bit for bit."""
    rng = np.random.default_rng(1)
    n = 200
    means = np.stack([rng.uniform(-1, 1, n), rng.uniform(-0.3, 0.3, n), rng.uniform(-0.5, 0.5, n)], 1)
    fld = field_from(means, np.exp(rng.normal(-2.5, 0.3, (n, 3))), rng.normal(size=(n, 4)),
                     rng.uniform(0.2, 0.9, n), rng.uniform(0, 1, (n, 3)), rng.uniform(0, 1, n))
    cam = synth.look_at([-3.0, 0.0, 0.0], [0.0, 0.0, 0.0], 64, 48, 60.0)
    start, centres, bins = np.array([0, n]), np.array([[0.0, 0.0, 0.0]]), [8]
    a = co.render_view_cached(fld, cam, start, bins, centres)
    b = oracle.render_view(fld, cam)
    assert a["order"][0] == np.argmin(fld.planes[0, :, 0]) and np.array_equal(a["rgbu"], b["rgbu"])


def test_cached_tiles_visited_front_to_back():
    """Two tiles split at x = 0 (tile 0: x < 0, tile 1: x >= 0) seen along +x
    from x = -3: tiles visited front to back (tile 0 first) with each tile in
    its bin-0 order give the global depth order, so the render equals the
    exact-sort render bit for bit -- the tiles overlap on screen, so visiting
    them back to front would not."""
    rng = np.random.default_rng(2)
    n = 240
    x = np.sort(rng.uniform(-1, 1, n))
    means = np.stack([x, rng.uniform(-0.3, 0.3, n), rng.uniform(-0.4, 0.4, n)], 1)
    fld = field_from(means, np.exp(rng.normal(-2.3, 0.3, (n, 3))), rng.normal(size=(n, 4)),
                     rng.uniform(0.3, 0.9, n), rng.uniform(0, 1, (n, 3)), rng.uniform(0, 1, n))
    split = int(np.searchsorted(x, 0.0))
    start = np.array([0, split, n])
    centres = np.array([[-0.5, 0.0, 0.0], [0.5, 0.0, 0.0]])
    cam = synth.look_at([-3.0, 0.0, 0.0], [0.0, 0.0, 0.0], 64, 48, 60.0)
    a = co.render_view_cached(fld, cam, start, [8, 8], centres)
    b = oracle.render_view(fld, cam)
    assert 0 < split < n and np.array_equal(a["rgbu"], b["rgbu"])


def test_cached_vs_exact_fidelity_on_flyover():
    """nearest-bin cached order vs exact per-frame depth sort, mean
    per-pixel |RGB| difference <= 0.02 on the default fly-over scene at 8
    bins (configs[3] geometry, 4,000 Gaussians per tile, 3 views)."""
    fld = synth.gen_config4_field(4_000)
    start, centres = synth.config4_tiles(4_000)
    bins = [co.bins_for(u) for u in co.tile_mean_uncertainty(fld, start)]
    assert set(bins) == {8}
    cams = synth.with_resolution(synth.flyover_cameras(64, 1920, 1080, 1500.0)[::21], 480, 270, 375.0)
    for cam in cams:
        a = co.render_view_cached(fld, cam, start, bins, centres)
        b = oracle.render_view(fld, cam)
        d = np.abs(a["rgbu"][..., :3] - b["rgbu"][..., :3]).mean()
        assert d <= 0.02, d
        assert not np.array_equal(a["rgbu"], b["rgbu"])  # approximate, not the exact order
