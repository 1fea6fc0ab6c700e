"""Pins of the CPU oracle against what the mathematics fixes (not against itself).

SURVEY.md §8(c) "What pins each part".  The paper prints no rasterizer values
(figures are placeholders), so each oracle function is
pinned by a closed form, a brute-force route, a library routine or an
invariant chosen so that a dropped term, wrong sign/index or transposed
operand fails at least one test.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle
import synth
from tests.helpers import axis_camera, field_from, random_unit_quats

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALPHA_MIN = np.float32(1.0) / np.float32(255.0)


# ----------------------------------------------------------------------------- exp_spec
def test_exp_spec_relative_error_vs_libm():
    """exp_spec within 1.2e-7 relative of exp (float64 libm) on [-80, 0]."""
    x = np.concatenate([np.linspace(-80.0, 0.0, 40001, dtype=np.float32),
                        np.float32([-1e-30, -1e-7, -0.5, -1.0, -np.log(255.0), -79.999])])
    got = oracle.exp_spec(x).astype(np.float64)
    ref = np.exp(x.astype(np.float64))
    rel = np.abs(got - ref) / ref
    assert rel.max() < 1.2e-7, rel.max()
    assert oracle.exp_spec(np.float32([0.0]))[0] == 1.0
    assert oracle.exp_spec(np.float32([-80.5, -1000.0])).tolist() == [0.0, 0.0]


# ----------------------------------------------------------------------------- SH basis
def _sphere_quadrature(nz=10, nphi=24):
    z, wz = np.polynomial.legendre.leggauss(nz)  # exact for polynomials in z up to 2nz-1
    phi = 2 * np.pi * np.arange(nphi) / nphi
    Z, PHI = np.meshgrid(z, phi, indexing="ij")
    W = np.outer(wz, np.full(nphi, 2 * np.pi / nphi))
    rho = np.sqrt(1 - Z ** 2)
    d = np.stack([rho * np.cos(PHI), rho * np.sin(PHI), Z], -1).reshape(-1, 3)
    return d, W.reshape(-1)


def test_sh_basis_orthonormal_and_addition_theorem():
    """Y_1..Y_15 are orthonormal on the sphere (exact quadrature) and obey the
    addition theorem sum_m Y_lm^2 = (2l+1)/(4 pi); Y_0 = 1 (DC = base colour)."""
    d, w = _sphere_quadrature()
    Y = np.array([oracle.sh_basis(di.astype(np.float32)) for di in d], dtype=np.float64)
    assert np.all(Y[:, 0] == 1.0)
    G = (Y[:, 1:] * w[:, None]).T @ Y[:, 1:]
    assert np.abs(G - np.eye(15)).max() < 2e-6
    for l in (1, 2, 3):
        s = (Y[:, l * l:(l + 1) ** 2] ** 2).sum(1)
        assert np.abs(s - (2 * l + 1) / (4 * np.pi)).max() < 2e-6


def test_sh_basis_matches_scipy_real_harmonics():
    """Library pin: Y_lm = sqrt(2) Re Y_l^m (m > 0), Y_l^0, sqrt(2) Im Y_l^|m| (m < 0),
    built from scipy's complex harmonics (Condon-Shortley phase included),
    ordered l = 1..3, m = -l..l -- fixes every sign of the pinned basis."""
    from scipy.special import sph_harm_y
    rng = np.random.default_rng(5)
    d = rng.normal(size=(64, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    for di in d.astype(np.float32):
        x, y, z = di.astype(np.float64)
        th, ph = math.acos(max(-1.0, min(1.0, z))), math.atan2(y, x)
        ref = [1.0]
        for l in (1, 2, 3):
            for m in range(-l, l + 1):
                c = sph_harm_y(l, abs(m), th, ph)
                ref.append(c.real if m == 0 else math.sqrt(2) * (c.real if m > 0 else c.imag))
        np.testing.assert_allclose(oracle.sh_basis(di), ref, rtol=0, atol=5e-6)


def test_sh_degree1_signs():
    """Degree-1 real SH with the Condon-Shortley phase: (-C1 y, C1 z, -C1 x)."""
    c1 = math.sqrt(3 / (4 * math.pi))
    for d in ([1, 0, 0], [0, 1, 0], [0, 0, 1]):
        Y = oracle.sh_basis(np.float32(d))
        np.testing.assert_allclose(Y[1:4], [-c1 * d[1], c1 * d[2], -c1 * d[0]], rtol=1e-7, atol=1e-8)


# ----------------------------------------------------------------------------- projection
def _cov_from_conic(p):
    M = np.array([[p["A"], p["B"]], [p["B"], p["C"]]], dtype=np.float64)
    return np.linalg.inv(M)


def test_projection_isotropic_on_axis_closed_form():
    """An isotropic sigma at depth D on the optical axis projects to
    Sigma' = ((f sigma / D)^2 + 0.3) I centred at (cx, cy) for ANY rotation."""
    rng = np.random.default_rng(1)
    f, D, sig = 100.0, 2.0, 0.05
    cam = axis_camera(64, 64, f)
    q = random_unit_quats(rng, 5)
    fld = field_from(np.tile([0, 0, D], (5, 1)), np.full((5, 3), sig), q, np.full(5, 0.7),
                     np.tile([0.2, 0.4, 0.6], (5, 1)), np.full(5, 0.5))
    P = oracle.project(fld, cam)
    s2 = (f * sig / D) ** 2 + 0.3
    for p in P:
        assert p["n_tiles"] > 0
        assert p["u"] == np.float32(32.0) and p["v"] == np.float32(32.0)
        cov = _cov_from_conic(p)
        np.testing.assert_allclose(np.diag(cov), [s2, s2], rtol=2e-6)
        assert abs(cov[0, 1]) < 1e-5 * s2
        assert p["depth_bits"] == np.float32(D).view(np.uint32)
        np.testing.assert_allclose([p["r"], p["g"], p["b"]], [0.2, 0.4, 0.6], rtol=1e-7)
        assert p["o"] == np.float32(0.7) and p["unc"] == np.float32(0.5)


def test_projection_distance_halves_radius():
    """Pinhole similar triangles: at 2x distance sqrt(Sigma' - 0.3 I) halves."""
    f, sig = 120.0, 0.04
    cam = axis_camera(64, 64, f)
    fld = field_from([[0, 0, 1.5], [0, 0, 3.0]], np.full((2, 3), sig), [[1, 0, 0, 0]] * 2, [0.5, 0.5],
                     [[1, 1, 1]] * 2, [1, 1])
    P = oracle.project(fld, cam)
    r1 = math.sqrt(_cov_from_conic(P[0])[0, 0] - 0.3)
    r2 = math.sqrt(_cov_from_conic(P[1])[0, 0] - 0.3)
    assert abs(r1 / r2 - 2.0) < 1e-5


def test_projection_matches_finite_difference_jacobian():
    """Sigma' - 0.3 I = J Sigma J^T with J the finite-difference Jacobian of the
    pinhole map p -> (fx x/z + cx, fy y/z + cy), Sigma from scipy's
    quaternion -> rotation matrix; within 1e-4 relative."""
    rng = np.random.default_rng(7)
    cam = synth.look_at([1.3, 2.1, -2.4], [0.1, -0.2, 0.05], 200, 160, 180.0)
    R = cam["R"].astype(np.float64).reshape(3, 3)
    t = cam["t"].astype(np.float64)
    f = float(cam["fx"])
    cx, cy = float(cam["cx"]), float(cam["cy"])

    def pix(p):
        c = R @ p + t
        return np.array([f * c[0] / c[2] + cx, f * c[1] / c[2] + cy])

    n = 12
    means = rng.uniform(-0.3, 0.3, (n, 3))
    scales = np.exp(rng.normal(-3.0, 0.5, (n, 3)))
    q = random_unit_quats(rng, n)
    fld = field_from(means, scales, q, np.full(n, 0.8), np.full((n, 3), 0.5), np.full(n, 0.5))
    P = oracle.project(fld, cam)
    m32 = fld.pos_opacity[:, :3].astype(np.float64)
    s32 = fld.scale_unc[:, :3].astype(np.float64)
    q32 = fld.rot.astype(np.float64)
    for i in range(n):
        assert P[i]["n_tiles"] > 0
        Rq = Rotation.from_quat([q32[i, 1], q32[i, 2], q32[i, 3], q32[i, 0]]).as_matrix()
        S3 = Rq @ np.diag(s32[i] ** 2) @ Rq.T
        h = 1e-5
        J = np.stack([(pix(m32[i] + h * e) - pix(m32[i] - h * e)) / (2 * h) for e in np.eye(3)], 1)
        ref = J @ S3 @ J.T
        got = _cov_from_conic(P[i]) - 0.3 * np.eye(2)
        assert np.abs(got - ref).max() < 1e-4 * np.abs(ref).max() + 1e-6, (i, got, ref)
        np.testing.assert_allclose([P[i]["u"], P[i]["v"]], pix(m32[i]), rtol=1e-6)


def test_projection_culls():
    """Behind / inside the near plane -> culled sentinel n_tiles = 0;
    off-screen -> n_tiles = 0."""
    cam = axis_camera(32, 32, 40.0)
    fld = field_from([[0, 0, -1.0], [0, 0, 0.2], [0, 0, 0.19], [50, 0, 1.0], [0, 0, 0.21]],
                     np.full((5, 3), 0.01), [[1, 0, 0, 0]] * 5, [0.5] * 5, [[1, 1, 1]] * 5, [1] * 5)
    P = oracle.project(fld, cam)
    assert P["n_tiles"].tolist()[:4] == [0, 0, 0, 0]
    assert P["n_tiles"][4] > 0


def _span_test_gaussians(rng, cam, trials):
    """Single Gaussians of every shape the spans must handle: tiny to large,
    strongly anisotropic (one thin axis), any rotation, any opacity, centred
    on and off screen."""
    for trial in range(trials):
        m = rng.uniform(-1.0, 1.0, (1, 3))
        s = np.exp(rng.normal(-2.5, 0.9, (1, 3)))
        if trial % 3 == 0:
            s[0, rng.integers(0, 3)] *= 0.05
        yield field_from(m, s, random_unit_quats(rng, 1), [rng.uniform(0.02, 1.0)], [[1, 1, 1]], [1])


def _alpha64(p, W, H):
    """float64 alpha = o exp(-q/2) at every pixel centre from the projected
    conic (the conic itself is pinned by the projection tests above)."""
    ys, xs = np.mgrid[0:H, 0:W]
    dx = float(p["u"]) - (xs + 0.5)
    dy = float(p["v"]) - (ys + 0.5)
    q = float(p["A"]) * dx * dx + 2.0 * float(p["B"]) * dx * dy + float(p["C"]) * dy * dy
    return float(p["o"]) * np.exp(-0.5 * q), q


def test_spans_contain_every_visible_pixel():
    """Lossless tiling (O1 step 15): every pixel whose alpha >= 1/255
    -- in the brute-force composite AND in float64 real arithmetic from the
    conic -- lies in a tile the Gaussian's spans emit."""
    rng = np.random.default_rng(3)
    cam = synth.look_at([0.0, 0.3, -3.0], [0, 0, 0], 72, 56, 70.0)
    W, H = 72, 56
    n_vis = 0
    for fld in _span_test_gaussians(rng, cam, 120):
        p = oracle.project(fld, cam)
        img = oracle.composite_brute(p, cam)
        ys, xs = np.nonzero(img["n_contrib"])
        if p[0]["n_tiles"] == 0:
            assert len(xs) == 0
            continue
        n_vis += 1
        tiles = set(oracle.tiles_of(p[0], cam))
        assert len(tiles) == int(p[0]["n_tiles"])
        assert all((y // 16, x // 16) in tiles for y, x in zip(ys, xs))
        a64, _ = _alpha64(p[0], W, H)
        ys, xs = np.nonzero(a64 >= (1.0 / 255.0) * (1.0 - 1e-6))
        assert all((y // 16, x // 16) in tiles for y, x in zip(ys, xs))
    assert n_vis > 60


def test_spans_are_tight():
    """Every emitted tile holds a pixel centre within (m + 1e-3) px of the
    ellipse q <= 11.1: q64 <= (sqrt(11.1) + (m + 1e-3) / sqrt(lambda_min(Sigma')))^2
    (float64 eigenvalues of the covariance = inverse conic).  Tiles of the
    3.33-sigma square box that only the box reaches are not emitted."""
    rng = np.random.default_rng(4)
    cam = synth.look_at([0.2, 0.5, -2.6], [0, 0, 0], 80, 64, 75.0)
    W, H = 80, 64
    saved = 0
    for fld in _span_test_gaussians(rng, cam, 120):
        p = oracle.project(fld, cam)[0]
        if p["n_tiles"] == 0:
            continue
        conic = np.array([[p["A"], p["B"]], [p["B"], p["C"]]], dtype=np.float64)
        lam_min = np.linalg.eigvalsh(np.linalg.inv(conic))[0]
        qmax = (math.sqrt(11.1) + (0.0625 + 1e-3) / math.sqrt(lam_min)) ** 2
        _, q = _alpha64(p, W, H)
        for ty, tx in oracle.tiles_of(p, cam):
            assert q[16 * ty:16 * ty + 16, 16 * tx:16 * tx + 16].min() <= qmax, (ty, tx)
        # the square box of radius ceil(3.33 sqrt(lambda_max))
        r = math.ceil(3.33 * math.sqrt(np.linalg.eigvalsh(np.linalg.inv(conic))[1]))
        bx = (min(max(math.floor((p["u"] - r) / 16), 0), 5), min(max(math.ceil((p["u"] + r) / 16), 0), 5))
        by = (min(max(math.floor((p["v"] - r) / 16), 0), 4), min(max(math.ceil((p["v"] + r) / 16), 0), 4))
        box = (bx[1] - bx[0]) * (by[1] - by[0])
        assert p["n_tiles"] <= box
        saved += box - int(p["n_tiles"])
    assert saved > 0


# ----------------------------------------------------------------------------- keys / sort / ranges
def _small_batch(seed=0, n=400, W=48, H=40, views=3, deg=1):
    fld, cams = synth.random_scene_small(seed, n, W, H, 50.0, views, deg)
    projs = [oracle.project(fld, c) for c in cams]
    return fld, cams, projs


def test_keys_emission_brute_force_enumeration():
    """O2 emission equals a brute-force enumeration over all (view, g, tile)
    triples of the batch grid, tested against each tile's membership in the
    Gaussian's spans; key = (view*gx*gy + ty*gx + tx) << 32 | depth bits."""
    fld, cams, projs = _small_batch()
    gx, gy = oracle.grid(cams[0])
    bs = oracle.bin_sort_batch(projs, cams)
    exp_k, exp_v = [], []
    for v, p in enumerate(projs):
        for g in range(len(p)):
            if p[g]["n_tiles"] == 0:
                continue
            member = set(oracle.tiles_of(p[g], cams[v]))
            for tile in range(gx * gy):
                ty, tx = divmod(tile, gx)
                if (ty, tx) in member:
                    exp_k.append(((v * gx * gy + tile) << 32) | int(p[g]["depth_bits"]))
                    exp_v.append(g)
    assert bs["keys_unsorted"].tolist() == exp_k
    assert bs["vals_unsorted"].tolist() == exp_v
    assert sum(int(p["n_tiles"].sum()) for p in projs) == len(exp_k)


def test_sort_and_ranges_invariants_vs_numpy():
    """O3: sorted list = numpy lexsort by (key, value); keys non-decreasing, equal
    keys have ascending values; ranges partition [0, K) and every key in a
    range carries that range's (view, tile)."""
    fld, cams, projs = _small_batch(seed=5, n=600)
    bs = oracle.bin_sort_batch(projs, cams)
    k, v = bs["keys_unsorted"], bs["vals_unsorted"]
    order = np.lexsort((v, k))
    assert np.array_equal(bs["keys"], k[order]) and np.array_equal(bs["vals"], v[order])
    sk, sv = bs["keys"], bs["vals"]
    assert np.all(sk[1:] >= sk[:-1])
    eq = sk[1:] == sk[:-1]
    assert np.all(sv[1:][eq] > sv[:-1][eq])
    rg = bs["ranges"].astype(np.int64)
    assert rg[0, 0] == 0 and rg[-1, 1] == len(sk)
    assert np.all(rg[1:, 0] == rg[:-1, 1]) and np.all(rg[:, 1] >= rg[:, 0])
    for t in range(len(rg)):
        seg = sk[rg[t, 0]:rg[t, 1]]
        assert np.all((seg >> np.uint64(32)) == t)
        d = (seg & np.uint64(0xFFFFFFFF)).view(np.uint64)
        assert np.all(d[1:] >= d[:-1])


def test_sort_adversarial_keys_vs_numpy():
    """qsort-based O3 on adversarial inputs: all-equal keys, extremes, top-digit-only."""
    rng = np.random.default_rng(0)
    cases = [
        (np.zeros(1000, np.uint64), rng.permutation(1000).astype(np.uint32)),
        (np.array([0, 2 ** 64 - 1, 5, 2 ** 64 - 1, 0], np.uint64), np.array([4, 3, 2, 1, 0], np.uint32)),
        ((rng.integers(0, 256, 3000).astype(np.uint64) << np.uint64(56)), rng.integers(0, 2 ** 32, 3000, dtype=np.uint64).astype(np.uint32)),
        (np.zeros(0, np.uint64), np.zeros(0, np.uint32)),
        (np.array([7], np.uint64), np.array([9], np.uint32)),
    ]
    for k, v in cases:
        sk, sv = oracle.sort_pairs(k, v)
        o = np.lexsort((v, k))
        assert np.array_equal(sk, k[o]) and np.array_equal(sv, v[o])


# ----------------------------------------------------------------------------- composite
def test_single_isotropic_gaussian_closed_form():
    """pixel = min(0.99, o exp(-rho^2 / (2 s^2))) (rgb, u) where alpha >= 1/255,
    else 0, with s^2 = (f sigma / D)^2 + 0.3 (float64 libm exp); score = mean U."""
    f, D, sig = 60.0, 2.5, 0.12
    for o in (0.99, 0.6, 0.03):
        cam = axis_camera(40, 36, f, cx=20.3, cy=17.8)
        rgb, unc = [0.3, 0.6, 0.9], 0.7
        fld = field_from([[0, 0, D]], [[sig] * 3], [[0.3, 0.5, -0.2, 0.6]], [o], [rgb], [unc])
        out = oracle.render_view(fld, cam)
        s2 = (f * sig / D) ** 2 + 0.3
        ys, xs = np.mgrid[0:36, 0:40]
        rho2 = (xs + 0.5 - 20.3) ** 2 + (ys + 0.5 - 17.8) ** 2
        a = np.minimum(0.99, np.float32(o) * np.exp(-0.5 * rho2 / s2))
        keep = a >= float(ALPHA_MIN)
        amb = np.abs(a - float(ALPHA_MIN)) < 1e-6
        exp = np.where(keep[..., None], a[..., None] * np.array(rgb + [unc]), 0.0)
        got = out["rgbu"].astype(np.float64)
        ok = ~amb
        assert np.abs(got - exp)[ok].max() < 1e-6
        assert np.array_equal(out["n_contrib"][ok] == 1, keep[ok])
        assert abs(out["score"] - got[..., 3].mean()) < 1e-12
        assert abs(out["score"] - exp[..., 3].mean()) < 1e-6


def test_single_anisotropic_gaussian_closed_form():
    """Image of one anisotropic Gaussian = o exp(-d^T Sigma'^-1 d / 2) clamped,
    with Sigma' = J Sigma J^T + 0.3 I from the finite-difference Jacobian and
    scipy's rotation (float64), within 2e-6 away from the 1/255 threshold."""
    rng = np.random.default_rng(21)
    cam = synth.look_at([0.4, 0.9, -2.5], [0.0, 0.1, 0.0], 64, 48, 60.0)
    R = cam["R"].astype(np.float64).reshape(3, 3)
    t = cam["t"].astype(np.float64)
    f, cx, cy = float(cam["fx"]), float(cam["cx"]), float(cam["cy"])

    def pix(p):
        c = R @ p + t
        return np.array([f * c[0] / c[2] + cx, f * c[1] / c[2] + cy])

    for trial in range(6):
        m = rng.uniform(-0.2, 0.2, (1, 3))
        s = np.array([[0.15, 0.03, 0.06]]) * rng.uniform(0.7, 1.3, (1, 3))
        q = random_unit_quats(rng, 1)
        fld = field_from(m, s, q, [0.9], [[0.5, 0.25, 1.0]], [0.8])
        out = oracle.render_view(fld, cam)
        m32 = fld.pos_opacity[0, :3].astype(np.float64)
        s32 = fld.scale_unc[0, :3].astype(np.float64)
        q32 = fld.rot[0].astype(np.float64)
        Rq = Rotation.from_quat([q32[1], q32[2], q32[3], q32[0]]).as_matrix()
        h = 1e-5
        J = np.stack([(pix(m32 + h * e) - pix(m32 - h * e)) / (2 * h) for e in np.eye(3)], 1)
        Sig = J @ (Rq @ np.diag(s32 ** 2) @ Rq.T) @ J.T + 0.3 * np.eye(2)
        Si = np.linalg.inv(Sig)
        mu = pix(m32)
        ys, xs = np.mgrid[0:48, 0:64]
        d = np.stack([xs + 0.5 - mu[0], ys + 0.5 - mu[1]], -1)
        qf = np.einsum("...i,ij,...j->...", d, Si, d)
        a = np.minimum(0.99, np.float32(0.9) * np.exp(-0.5 * qf))
        keep = a >= float(ALPHA_MIN)
        ok = np.abs(a - float(ALPHA_MIN)) > 1e-5
        exp = np.where(keep, a, 0.0)
        assert np.abs(out["rgbu"][..., 3] - 0.8 * exp)[ok].max() < 2e-6
        assert np.abs(out["rgbu"][..., 2] - exp)[ok].max() < 2e-6


def test_two_gaussians_front_half_over_opaque():
    """0.5 in front of an opaque Gaussian -> 0.5 c_f + 0.495 c_b (S:L120 with the
    0.99 alpha clamp), at a pixel centre sitting exactly on both means."""
    cam = axis_camera(17, 17, 50.0, cx=8.5, cy=8.5)
    cf, cb = [0.8, 0.1, 0.3], [0.2, 0.9, 0.5]
    fld = field_from([[0, 0, 1.0], [0, 0, 2.0]], [[0.05] * 3] * 2, [[1, 0, 0, 0]] * 2, [0.5, 1.0],
                     [cf, cb], [0.25, 0.75])
    out = oracle.render_view(fld, cam)
    px = out["rgbu"][8, 8].astype(np.float64)
    exp = 0.5 * np.array(cf + [0.25]) + 0.495 * np.array(cb + [0.75])
    np.testing.assert_allclose(px, exp, atol=1e-6)
    assert out["n_contrib"][8, 8] == 2
    np.testing.assert_allclose(out["t_final"][8, 8], 0.005, rtol=1e-6)


def test_termination_stops_before_blending():
    """T stop rule: the Gaussian that would take T below 1e-4 is NOT blended,
    so T_final >= 1e-4 (three alpha=0.99 layers: T 1 -> 0.01 -> 1e-4 -> stop)."""
    cam = axis_camera(17, 17, 50.0, cx=8.5, cy=8.5)
    # layers alpha 0.99, 0.99, 0.5: float32 T after layer 1 is 1 - 0.99f; layer 2
    # would give T1 * (1 - 0.99f) < 1e-4 -> stop.  Layer 3 (alpha 0.5) would keep
    # T above 1e-4 but must not be reached: the loop ends at the first stop.
    fld = field_from([[0, 0, 1.0], [0, 0, 1.5], [0, 0, 2.0]], [[0.05] * 3] * 3, [[1, 0, 0, 0]] * 3,
                     [1.0, 1.0, 0.5], [[1, 0, 0], [0, 1, 0], [0, 0, 1]], [1, 1, 1])
    out = oracle.render_view(fld, cam)
    T1 = np.float32(1) - np.float32(0.99)
    assert T1 * T1 < np.float32(1e-4) <= T1 * np.float32(0.5)
    assert out["n_contrib"][8, 8] == 1
    assert out["t_final"][8, 8] == T1
    np.testing.assert_allclose(out["rgbu"][8, 8], [0.99, 0, 0, 0.99], rtol=1e-7)


def test_termination_threshold_closed_form():
    """The 1e-4 stop threshold itself (O5): a stack of eight identical layers
    centred on a pixel, each alpha = 0.8 there (exp(0) = 1 exactly, o = 0.8),
    blends exactly k = floor(ln 1e-4 / ln 0.2) = 5 layers (0.2^5 = 3.2e-4 >=
    1e-4 > 0.2^6 = 6.4e-5, both far from the threshold), T_final = 0.2^5,
    U = 1 - 0.2^5.  A threshold of 1e-3 would stop after 4, of 1e-5 after 7."""
    k = int(np.floor(np.log(1e-4) / np.log(0.2)))
    assert k == 5 and 0.2 ** k > 1e-3 / 4 and 0.2 ** (k + 1) < 1e-4
    cam = axis_camera(17, 17, 50.0, cx=8.5, cy=8.5)
    n = 8
    fld = field_from([[0, 0, 1.0 + 0.25 * i] for i in range(n)], [[0.05] * 3] * n, [[1, 0, 0, 0]] * n,
                     [0.8] * n, [[0, 0, 0]] * n, [1] * n)
    out = oracle.render_view(fld, cam)
    assert out["n_contrib"][8, 8] == k
    np.testing.assert_allclose(out["t_final"][8, 8], 0.2 ** k, rtol=1e-5)
    np.testing.assert_allclose(out["rgbu"][8, 8, 3], 1.0 - 0.2 ** k, rtol=1e-5)


@pytest.mark.parametrize("seed,deg", [(0, 0), (1, 1), (2, 2), (3, 3), (4, 3)])
def test_brute_force_equals_tiled_bit_exact(seed, deg):
    """Tiled (per-tile sorted lists) == brute force (all Gaussians, global depth
    order) bit for bit: pixels outside a Gaussian's spans take the alpha < 1/255
    skip, so both loops perform identical state updates.  48x40 image = 3x3 tiles
    with ragged right/bottom tiles."""
    fld, cams = synth.random_scene_small(seed, 300, 48, 40, 45.0, 2, deg, logscale_mu=-2.2)
    for cam in cams:
        p = oracle.project(fld, cam)
        t = oracle.render_view(fld, cam)
        b = oracle.composite_brute(p, cam)
        assert t["n_frag"] > 0
        for key in ("rgbu", "t_final", "n_contrib"):
            assert np.array_equal(t[key], b[key]), key
        assert t["score"] == b["score"]


@pytest.mark.parametrize("u,probe,visible", [(17.0, 32, True), (31.0, 48, False)])
def test_edge_aligned_box_is_lossless(u, probe, visible):
    """SURVEY §8(c) k row: isotropic Sigma' = 25 I, o = 0.99.  At u = 17 a
    k = 3 box (r = 15) would stop at pixel 31 but pixel 32 has alpha = 0.0081 >=
    1/255; the q <= 11.1 spans (x-extent 16.66 px) keep it.  At u = 31 pixel 48
    (first pixel past the span, tile 3) has alpha = 0.0022 < 1/255."""
    f, D = 100.0, 2.0
    sig = D * math.sqrt(24.7) / f
    cam = axis_camera(80, 16, f, cx=u, cy=8.5)
    fld = field_from([[0, 0, D]], [[sig] * 3], [[1, 0, 0, 0]], [0.99], [[1, 1, 1]], [1.0])
    p = oracle.project(fld, cam)
    t = oracle.render_view(fld, cam)
    b = oracle.composite_brute(p, cam)
    assert np.array_equal(t["rgbu"], b["rgbu"])
    rho = probe + 0.5 - u
    a = 0.99 * math.exp(-0.5 * rho * rho / 25.0)
    assert (a >= 1 / 255) == visible
    assert (t["n_contrib"][8, probe] == 1) == visible
    if visible:
        assert abs(t["rgbu"][8, probe, 3] - a) < 1e-5


def test_compositing_invariants_and_uniform_uncertainty():
    """T_final in [1e-4, 1]; n_contrib <= list length; with every u = 1 the
    U channel equals sum w = 1 - T_final (to float rounding); U <= max u (1 - T_final)."""
    sc = synth.make_scene(1, n_override=3000, views=2)
    fld = sc.field
    fld.planes[1, :, 3] = 1.0
    for cam in sc.cameras:
        out = oracle.render_view(fld, cam)
        tf, U = out["t_final"], out["rgbu"][..., 3]
        assert np.all(tf >= np.float32(1e-4)) and np.all(tf <= 1.0)
        assert np.abs(U - (1.0 - tf)).max() < 2e-6
        gx, _ = oracle.grid(cam)
        ys, xs = np.mgrid[0:cam["height"], 0:cam["width"]]
        tile = (ys // 16) * gx + xs // 16
        rg = out["ranges"].astype(np.int64)
        assert np.all(out["n_contrib"] <= (rg[tile, 1] - rg[tile, 0]))
        assert np.all(out["rgbu"][..., :3] >= 0)


def test_score_linear_in_uncertainty_and_bounded():
    """score(2u) == 2 score(u) exactly (power-of-two scaling commutes with every
    rounding); 0 <= score <= max u."""
    sc = synth.make_scene(1, n_override=2000, views=1)
    cam = sc.cameras[0]
    s1 = oracle.render_view(sc.field, cam)["score"]
    f2 = synth.GaussianField(sc.field.planes.copy(), 0)
    f2.planes[1, :, 3] *= 2
    s2 = oracle.render_view(f2, cam)["score"]
    assert s2 == 2 * s1
    assert 0 <= s1 <= sc.field.planes[1, :, 3].max()


def test_permutation_invariance_and_determinism():
    """Permuting Gaussian indices leaves the image bit-identical when no two
    Gaussians share a depth; two runs are bit-identical."""
    sc = synth.make_scene(1, n_override=2000, views=1)
    cam = sc.cameras[0]
    a = oracle.render_view(sc.field, cam)
    a2 = oracle.render_view(sc.field, cam)
    assert np.array_equal(a["rgbu"], a2["rgbu"])
    d = a["proj"]["depth_bits"][a["proj"]["n_tiles"] > 0]
    assert len(np.unique(d)) == len(d)
    perm = np.random.default_rng(0).permutation(sc.field.n)
    b = oracle.render_view(sc.field.subset(perm), cam)
    assert np.array_equal(a["rgbu"], b["rgbu"]) and a["score"] == b["score"]


def test_render_views_threaded_equals_single():
    sc = synth.make_scene(1, n_override=2000, views=4)
    scores, nf, nk, rgbu = oracle.render_views(sc.field, sc.cameras, n_threads=3, images=True)
    for i, cam in enumerate(sc.cameras):
        r = oracle.render_view(sc.field, cam)
        assert r["score"] == scores[i] and r["n_frag"] == nf[i] and len(r["keys"]) == nk[i]
        assert np.array_equal(r["rgbu"], rgbu[i])


# ----------------------------------------------------------------------------- NBV / top-k
def test_select_topk_golden_examples():
    g = json.load(open(os.path.join(GOLDEN, "select_topk.json")))
    for c in g["cases"]:
        assert oracle.select_topk(c["scores"], c["k"], c.get("exclude")).tolist() == c["expect"], c["cite"]
    for c in g["errors"]:
        with pytest.raises(ValueError):
            oracle.select_topk(c["scores"], c["k"], c.get("exclude"))


def test_select_topk_is_exhaustive_optimum():
    """Greedy top-k = argmax over all |V| = k subsets of the additive objective
    (App. A.2), for N <= 12, k <= 4."""
    rng = np.random.default_rng(11)
    for trial in range(30):
        n = int(rng.integers(5, 13))
        k = int(rng.integers(1, 5))
        s = rng.integers(0, 6, n) / 5.0  # many ties
        ex = rng.random(n) < 0.2
        avail = [i for i in range(n) if not ex[i]]
        if k > len(avail):
            continue
        sel = oracle.select_topk(s, k, ex)
        best = max(sum(s[list(c)]) for c in itertools.combinations(avail, k))
        assert abs(sum(s[sel]) - best) < 1e-12
        assert not ex[sel].any() and len(set(sel.tolist())) == k
        assert all(s[sel[i]] >= s[sel[i + 1]] for i in range(k - 1))
