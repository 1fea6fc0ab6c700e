"""Pins of the NEXT-2 LOD blending in the oracle (PAPER.md eq:lod_blend
L124-127, clamped form App. A.4; SPEC lod-cache S:L563-591):
printed examples, complementarity / partition of unity, the C0 Lipschitz
bound, and the rendering equivalences (w scales the opacity; o w < 1/255 is
culled)."""
import json
import math
import os

import numpy as np

import oracle
import synth
from tests.helpers import axis_camera, field_from

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "lod_examples.json")


def _lod(levels, thresholds, delta, tl=None):
    return synth.LodData(np.zeros((1, 4), np.float32) if tl is None else tl, levels, delta, tuple(thresholds))


def test_lod_golden_examples():
    g = json.load(open(GOLDEN))
    for c in g["blend"]:
        assert oracle.lod_blend(c["d"], c["D"], c["delta"]) == c["expect"], c["cite"]
    for c in g["levels"]:
        L = _lod(len(c["thresholds"]) + 1, c["thresholds"], c["delta"])
        got = [oracle.lod_weight(c["d"], l, L) for l in range(L.levels)]
        assert got == c["expect"], c["cite"]


def test_lod_partition_of_unity_and_lipschitz():
    """Levels partition the opacity: sum_l w_l(d) = 1 on a dense sweep (bands
    do not overlap: 2 delta < every gap); each w_l is C0 with slope <= 1/(2 delta)
    (App. A.4 'C0 continuous by construction', SPEC acceptance 9)."""
    L = _lod(6, (1.5, 3.0, 6.0, 12.0, 24.0), 0.25)
    d = np.linspace(0.0, 30.0, 10001)
    W = np.array([[oracle.lod_weight(x, l, L) for l in range(6)] for x in d])
    assert np.abs(W.sum(1) - 1.0).max() < 1e-6
    eps = d[1] - d[0]
    assert np.abs(np.diff(W, axis=0)).max() <= eps / (2 * 0.25) + 1e-6
    # inside band i exactly levels i and i+1 are active and complementary
    for i, D in enumerate(L.thresholds):
        x = D + 0.1
        w = [oracle.lod_weight(x, l, L) for l in range(6)]
        assert abs(w[i] + w[i + 1] - 1.0) < 1e-7 and sum(w) - w[i] - w[i + 1] == 0.0


def test_lod_weight_scales_opacity_in_render():
    """A level-1 Gaussian at weight w renders bit-identically to the same
    Gaussian with stored opacity float32(o w) and no LOD; at o w < 1/255 it is
    culled (n_tiles = 0, image 0)."""
    cam = axis_camera(48, 40, 60.0)
    D, delta, o = 2.0, 0.5, 0.8
    # camera at the origin, tile centre at distance d on the axis
    n_culled = 0
    for d in (2.0, 1.8, 2.3, 2.49, 2.497, 2.7):
        tl = np.array([[0.0, 0.0, d, 1.0]], np.float32)
        L = _lod(3, (1.0, D), delta, tl)
        w = oracle.lod_weight(np.float32(d), 1, L)
        fld = field_from([[0, 0, 2.0]], [[0.08] * 3], [[1, 0, 0, 0]], [o], [[0.3, 0.6, 0.9]], [0.5])
        a = oracle.render_view(fld, cam, L)
        if np.float32(o) * np.float32(w) < np.float32(1) / np.float32(255):
            assert a["proj"]["n_tiles"][0] == 0 and not a["rgbu"].any()
            n_culled += 1
            continue
        assert a["proj"]["n_tiles"][0] > 0
        ref = fld.planes.copy()
        ref[0, 0, 3] = np.float32(o) * np.float32(w)
        b = oracle.render_view(synth.GaussianField(ref, 0), cam)
        assert np.array_equal(a["rgbu"], b["rgbu"]) and a["score"] == b["score"]
        assert math.isclose(float(a["proj"]["o"][0]), o * w, rel_tol=1e-6)
    assert n_culled == 2


def test_lod_render_matches_brute_force_and_levels_sum():
    """LOD scene: tiled == brute force bit for bit (the cull keeps tiling
    lossless), and every visible opacity is the base opacity times the level
    weight at the camera's distance to the tile centre."""
    rng = np.random.default_rng(5)
    fld, cams = synth.random_scene_small(2, 300, 48, 40, 45.0, 2, 1, logscale_mu=-2.2)
    L = synth.random_lod(rng, fld.n)
    for cam in cams:
        p = oracle.project(fld, cam, L)
        t = oracle.render_view(fld, cam, L)
        b = oracle.composite_brute(p, cam)
        for key in ("rgbu", "t_final", "n_contrib"):
            assert np.array_equal(t[key], b[key]), key
        # opacities are the base opacities times the weights
        vis = p["n_tiles"] > 0
        campos = cam["campos"].astype(np.float32)
        for g in np.nonzero(vis)[0][:50]:
            c = L.tile_level[g]
            d = np.sqrt(np.float32(((campos[0] - c[0]) * (campos[0] - c[0]) + (campos[1] - c[1]) * (campos[1] - c[1]))
                                   + (campos[2] - c[2]) * (campos[2] - c[2])))
            assert p["o"][g] == np.float32(fld.planes[0, g, 3]) * np.float32(oracle.lod_weight(d, int(c[3]), L))
