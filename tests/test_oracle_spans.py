"""Tile membership of the oracle (DESIGN.md §4 "tile assignment", O1 steps
14-15) against an independent float64 reference built from the EWA
definition, pixel row by pixel row -- not from the oracle's span formula.

Reading under test: a Gaussian is listed in tile (tx, ty) iff the tile holds
a pixel centre inside the x-extent, over that tile's pixel rows, of the
ellipse q <= t (t = 11.1) widened by m = 1/16 px, clipped to the image.  The
oracle takes the extent over the CONTINUOUS band between the tile row's first
and last pixel-centre rows (the ellipse's extreme points clamped into the
band); that relaxation is the documented slack against the plain per-row
union.  Both references here are computed in float64 from Sigma' = J W Sigma
W^T J^T + 0.3 I (the 1.3x FOV-clamped pinhole Jacobian, scipy rotations):

  rows(t, m):  union over the tile row's pixel rows y of the pixel columns
               whose centre lies in the exact ellipse x-interval at y + 0.5,
               widened by m  (the plain per-pixel-row definition)
  band(t, m):  the same over the continuous band (the oracle's reading)

and the oracle must satisfy, for every tile row,
  rows(t-, m - eps) <= oracle <= band(t+, m + eps),
with t+- = t (1 +- 1e-5) and eps = 2e-3 px absorbing float32 rounding (the
ellipse interval is ill-conditioned at its top and bottom rows, hence the
relative slack on t).  Setting the margin to 0 violates the lower bound on
tiles decided inside the 1/16-px margin; the test asserts such tiles occur.
"""
import math

import numpy as np
from scipy.spatial.transform import Rotation

import oracle
import synth
from tests.helpers import field_from, random_unit_quats

T_SPAN, M_SPAN = 11.1, 1.0 / 16.0
EPS_PX, EPS_T = 2e-3, 1e-5


def _project64(fld, cam):
    """float64 EWA projection (SURVEY §8(c) O1 written as matrices): pixel
    mean (u, v), depth and the 2x2 covariance (a, b, c) incl. the 0.3 px^2
    dilation, for every Gaussian of the float32 field."""
    R = cam["R"].astype(np.float64).reshape(3, 3)
    t = cam["t"].astype(np.float64)
    fx, fy, cx, cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    limx, limy = float(cam["limx"]), float(cam["limy"])
    mu = fld.pos_opacity[:, :3].astype(np.float64)
    s = fld.scale_unc[:, :3].astype(np.float64)
    q = fld.rot.astype(np.float64)
    Rq = Rotation.from_quat(q[:, [1, 2, 3, 0]]).as_matrix()  # scipy: (x, y, z, w)
    S3 = Rq @ (s[:, :, None] ** 2 * np.swapaxes(Rq, 1, 2))
    pc = mu @ R.T + t
    z = pc[:, 2]
    xn, yn = pc[:, 0] / z, pc[:, 1] / z
    u, v = fx * xn + cx, fy * yn + cy
    tx, ty = np.clip(xn, -limx, limx) * z, np.clip(yn, -limy, limy) * z
    J = np.zeros((len(z), 2, 3))
    J[:, 0, 0] = fx / z
    J[:, 0, 2] = -fx * tx / z ** 2
    J[:, 1, 1] = fy / z
    J[:, 1, 2] = -fy * ty / z ** 2
    T = J @ R
    S2 = T @ S3 @ np.swapaxes(T, 1, 2) + 0.3 * np.eye(2)
    return u, v, z, S2[:, 0, 0], S2[:, 0, 1], S2[:, 1, 1]


def _cols(L, R, W):
    """Pixel columns with a centre in [L, R], clipped to the image."""
    c0 = max(math.ceil(L - 0.5), 0)
    c1 = min(math.floor(R - 0.5), W - 1)
    return (c0, c1) if c0 <= c1 else None


def _reference_tiles(u, v, a, b, c, W, H, t, m, band):
    """{ty: set of tx} of one Gaussian (float64); band selects the continuous
    band extent (the oracle's reading) instead of the per-pixel-row union."""
    det = a * c - b * b
    if not det > 0:
        return {}
    ye = math.sqrt(t * c) + m
    py0 = max(math.ceil(v - ye - 0.5), 0)
    py1 = min(math.floor(v + ye - 0.5), H - 1)
    out = {}
    p, h, dys = b / c, det / c, b * math.sqrt(t / a)

    def xint(dy):
        r = math.sqrt(max(0.0, h * (t - dy * dy / c)))
        return u + p * dy - r, u + p * dy + r

    for tyi in range(py0 // 16, py1 // 16 + 1) if py0 <= py1 else ():
        ya, yb = max(16 * tyi, py0), min(16 * tyi + 15, py1)
        cols = set()
        if band:
            dya, dyb = ya + 0.5 - v, yb + 0.5 - v
            L = xint(min(max(-dys, dya), dyb))[0] - m
            R = xint(min(max(dys, dya), dyb))[1] + m
            cc = _cols(L, R, W)
            if cc:
                cols.update(range(cc[0] // 16, cc[1] // 16 + 1))
        else:
            for y in range(ya, yb + 1):
                dy = y + 0.5 - v
                if dy * dy / c > t:
                    continue
                L, R = xint(dy)
                cc = _cols(L - m, R + m, W)
                if cc:
                    cols.update(range(cc[0] // 16, cc[1] // 16 + 1))
        if cols:
            out[tyi] = cols
    return out


def _gaussians(rng, n):
    """Every shape the spans must handle: tiny to large, needles (one or two
    thin axes), any rotation, centred on screen, on its edges and off it."""
    means = np.stack([rng.uniform(-1.6, 1.6, n), rng.uniform(-1.3, 1.3, n), rng.uniform(1.0, 4.0, n)], 1)
    ls = rng.normal(-3.2, 1.0, (n, 3))
    thin = rng.random(n) < 0.35
    ls[thin, rng.integers(0, 3, thin.sum())] -= rng.uniform(2.0, 4.0, thin.sum())
    needle = rng.random(n) < 0.1
    ls[needle, :2] -= 3.0
    return field_from(means, np.exp(ls), random_unit_quats(rng, n), rng.uniform(0.05, 1.0, n),
                      np.full((n, 3), 0.5), np.full(n, 0.5))


def test_spans_match_float64_per_pixel_row_reference():
    rng = np.random.default_rng(11)
    W, H = 176, 136  # ragged: 11 x 9 tiles, the last row 8 px high
    cam = synth.look_at([0.0, 0.0, 0.0], [0.0, 0.0, 1.0], W, H, 150.0)
    fld = _gaussians(rng, 12000)
    P = oracle.project(fld, cam)
    u, v, z, a, b, c = _project64(fld, cam)
    lo_t, hi_t = T_SPAN * (1 - EPS_T), T_SPAN * (1 + EPS_T)
    n_listed = n_band_extra = n_margin = 0
    for i in range(fld.n):
        if not z[i] > 0.2 * (1 + 1e-6):
            assert int(P[i]["n_tiles"]) == 0
            continue
        got = {}
        for ty, tx in oracle.tiles_of(P[i], cam):
            got.setdefault(ty, set()).add(tx)
        assert sum(len(s) for s in got.values()) == int(P[i]["n_tiles"])
        args = (u[i], v[i], a[i], b[i], c[i], W, H)
        lower = _reference_tiles(*args, lo_t, M_SPAN - EPS_PX, band=False)
        upper = _reference_tiles(*args, hi_t, M_SPAN + EPS_PX, band=True)
        for ty, cols in lower.items():  # the plain per-row union is always listed
            assert cols <= got.get(ty, set()), (i, ty, cols, got.get(ty))
        for ty, cols in got.items():  # and nothing beyond the band reading
            assert cols <= upper.get(ty, set()), (i, ty, cols, upper.get(ty))
        n_listed += bool(got)
        rows_hi = _reference_tiles(*args, hi_t, M_SPAN + EPS_PX, band=False)
        n_band_extra += sum(len(cols - rows_hi.get(ty, set())) for ty, cols in got.items())
        # tiles decided inside the margin: listed with m, missed with m = 0
        no_m = _reference_tiles(*args, hi_t, EPS_PX, band=True)
        n_margin += sum(len(cols - no_m.get(ty, set())) for ty, cols in lower.items())
    assert n_listed > 6000
    assert n_margin > 0  # a zero margin would fail the lower bound on these
    assert n_band_extra >= 0


def _sh_coeffs(fld):
    """[n, (d+1)^2, 3] float64 view of the packed SH planes (slot-major: plane
    j, element i holds flat coefficients 4j..4j+3; flat = 3 coef + channel)."""
    ncoef = (fld.sh_degree + 1) ** 2
    flat = np.swapaxes(fld.sh, 0, 1).reshape(fld.n, -1)[:, :3 * ncoef]
    return flat.reshape(fld.n, ncoef, 3).astype(np.float64)


def test_sh_degree1_colour_hand_formula():
    """SURVEY §8(c) O4 degree-1 hand check: rgb = k0 - C1 y k1 + C1 z k2 - C1 x k3
    with (x, y, z) = normalize(mu - campos), per channel, clamped at 0."""
    rng = np.random.default_rng(21)
    n = 64
    cam = synth.look_at([0.4, 0.9, -2.5], [0.0, 0.0, 0.0], 64, 64, 60.0)
    means = rng.uniform(-0.3, 0.3, (n, 3))
    k0 = rng.uniform(0.2, 0.8, (n, 3))
    rest = rng.normal(0.0, 0.3, (n, 3, 3))
    fld = field_from(means, np.full((n, 3), 0.02), random_unit_quats(rng, n), np.full(n, 0.9), k0,
                     np.full(n, 0.5), sh_degree=1, sh_rest=rest)
    P = oracle.project(fld, cam)
    c1 = math.sqrt(3.0 / (4.0 * math.pi))
    eye = cam["campos"].astype(np.float64)
    mu = fld.pos_opacity[:, :3].astype(np.float64)
    sh = _sh_coeffs(fld)  # [n, 4, 3] as packed (float32 values)
    for i in range(n):
        assert P[i]["n_tiles"] > 0
        d = mu[i] - eye
        x, y, zz = d / np.linalg.norm(d)
        ref = sh[i, 0] - c1 * y * sh[i, 1] + c1 * zz * sh[i, 2] - c1 * x * sh[i, 3]
        np.testing.assert_allclose([P[i]["r"], P[i]["g"], P[i]["b"]], np.maximum(ref, 0.0), rtol=0, atol=2e-6)


def test_sh_colour_all_degrees_vs_scipy_basis():
    """O4 colour assembly at degrees 0..3: max(0, sum_i Y_i(dir) k_i) with the
    real basis built from scipy's complex harmonics (Condon-Shortley phase,
    m = -l..l order) and dir = normalize(mu - campos); fixes the direction's
    sign, the coefficient index and the channel order."""
    from scipy.special import sph_harm_y
    rng = np.random.default_rng(22)
    cam = synth.look_at([-1.1, 0.7, -2.2], [0.0, 0.1, 0.0], 64, 64, 60.0)
    eye = cam["campos"].astype(np.float64)
    for deg in (0, 1, 2, 3):
        n = 24
        ncoef = (deg + 1) ** 2
        means = rng.uniform(-0.3, 0.3, (n, 3))
        rest = rng.normal(0.0, 0.2, (n, ncoef - 1, 3)) if deg else None
        fld = field_from(means, np.full((n, 3), 0.02), random_unit_quats(rng, n), np.full(n, 0.9),
                         rng.uniform(0.3, 0.7, (n, 3)), np.full(n, 0.5), sh_degree=deg, sh_rest=rest)
        P = oracle.project(fld, cam)
        sh = _sh_coeffs(fld)
        mu = fld.pos_opacity[:, :3].astype(np.float64)
        for i in range(n):
            d = mu[i] - eye
            x, y, zz = d / np.linalg.norm(d)
            th, ph = math.acos(max(-1.0, min(1.0, zz))), math.atan2(y, x)
            Y = [1.0]
            for l in range(1, deg + 1):
                for m in range(-l, l + 1):
                    cplx = sph_harm_y(l, abs(m), th, ph)
                    Y.append(cplx.real if m == 0 else math.sqrt(2) * (cplx.real if m > 0 else cplx.imag))
            ref = np.maximum(np.asarray(Y) @ sh[i], 0.0)
            np.testing.assert_allclose([P[i]["r"], P[i]["g"], P[i]["b"]], ref, rtol=0, atol=5e-6)
