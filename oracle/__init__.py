"""CPU oracle for the active-view scoring rasterizer -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2602_15355_b200``) never imports it, and this package
never imports the product path: the two share no code.  Inputs come from the
``synth`` module, which holds none of the method's arithmetic.

The arithmetic lives in ``gsr_oracle.c`` (plain C, float32, no implicit
contraction; see its header and SURVEY.md §8(c) O1-O7).  This file is ctypes
marshalling plus the top-k rule O7, written in plain Python.

Every function cites the passage it follows; the rasterizer constants are the
readings listed in DESIGN.md "Readings of the paper" (the paper itself prints
no rasterizer -- PAPER.md §3.5 L119-130 and Alg. 1 L146-154 only name the
steps).  Pins: tests/test_oracle_*.py.  Parity pinned for every function here
(no "parity unpinned" entries).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gsr_oracle.c")
# GSR_ORACLE_LIB: a prebuilt (e.g. deliberately mutated) oracle library, for
# scripts/oracle_mutants.py only; build() never overwrites it
_LIB = os.environ.get("GSR_ORACLE_LIB") or os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]

PROJ_DTYPE = np.dtype(
    [("u", "<f4"), ("v", "<f4"), ("A", "<f4"), ("B", "<f4"), ("C", "<f4"), ("o", "<f4"),
     ("unc", "<f4"), ("r", "<f4"), ("g", "<f4"), ("b", "<f4"),
     ("sp_p", "<f4"), ("sp_h", "<f4"), ("sp_ic", "<f4"), ("sp_dys", "<f4"),
     ("depth_bits", "<u4"), ("py0", "<u4"), ("py1", "<u4"), ("n_tiles", "<u4")])
assert PROJ_DTYPE.itemsize == 72

TILE = 16


class _Lod(ctypes.Structure):
    """orc_lod: NEXT-2 LOD blending parameters (PAPER.md eq:lod_blend)."""
    _fields_ = [("levels", ctypes.c_int32), ("delta", ctypes.c_float), ("thresholds", ctypes.c_float * 7),
                ("tile_level", ctypes.c_void_p)]


def _lod(lod):
    """(ctypes struct or None, keep-alive array) from a synth.LodData (or None)."""
    if lod is None:
        return None, None
    tl = np.ascontiguousarray(lod.tile_level, dtype=np.float32)
    th = (ctypes.c_float * 7)(*[float(x) for x in list(lod.thresholds) + [0.0] * (7 - len(lod.thresholds))])
    return _Lod(int(lod.levels), float(lod.delta), th, tl.ctypes.data), tl


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FMA contraction)."""
    if os.environ.get("GSR_ORACLE_LIB"):
        return _LIB
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm", "-lpthread"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        L.orc_exp_spec.argtypes = [ctypes.c_float]
        L.orc_exp_spec.restype = ctypes.c_float
        L.orc_sh_basis.argtypes = [ctypes.c_float] * 3 + [P]
        L.orc_project.argtypes = [P, i64, ctypes.c_int, P, P, P]
        L.orc_lod_blend.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_float]
        L.orc_lod_blend.restype = ctypes.c_float
        L.orc_lod_weight.argtypes = [ctypes.c_float, ctypes.c_int, P]
        L.orc_lod_weight.restype = ctypes.c_float
        L.orc_row_span.argtypes = [P, ctypes.c_uint32, ctypes.c_int, P, P]
        L.orc_count_keys.argtypes = [P, i64]
        L.orc_count_keys.restype = i64
        L.orc_emit_keys.argtypes = [P, i64, P, i32, P, P]
        L.orc_sort_pairs.argtypes = [P, P, i64]
        L.orc_emit_keys_order.argtypes = [P, P, i64, P, i32, P, P]
        L.orc_ranges.argtypes = [P, i64, i64, P]
        L.orc_composite_tiled.argtypes = [P, P, P, P, P, P, P, P]
        L.orc_composite_tiled.restype = ctypes.c_double
        L.orc_composite_brute.argtypes = [P, i64, P, P, P, P, P]
        L.orc_composite_brute.restype = ctypes.c_double
        L.orc_composite_trace.argtypes = [P, P, P, P, P, P, i64]
        L.orc_composite_trace.restype = i64
        L.orc_render_views.argtypes = [P, i64, ctypes.c_int, P, i32, P, ctypes.c_int, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _cam(cam):
    """One camera as a contiguous 1-element CAM_DTYPE array."""
    return np.ascontiguousarray(np.asarray(cam).reshape(1))


def _wh(cam):
    c = np.asarray(cam).reshape(-1)[0]
    return int(c["width"]), int(c["height"])


def grid(cam):
    W, H = _wh(cam)
    return (W + TILE - 1) // TILE, (H + TILE - 1) // TILE


# ---------------------------------------------------------------------------
def exp_spec(x):
    """SURVEY §8(c) O5 exp_spec, elementwise (float32 in, float32 out)."""
    L = lib()
    x = np.asarray(x, dtype=np.float32)
    return np.array([L.orc_exp_spec(float(v)) for v in x.reshape(-1)], dtype=np.float32).reshape(x.shape)


def sh_basis(d):
    """SURVEY §8(c) O4 real SH basis (Y0 = 1) at unit direction d (float32)."""
    L = lib()
    out = np.zeros(16, dtype=np.float32)
    L.orc_sh_basis(float(d[0]), float(d[1]), float(d[2]), _p(out))
    return out


def project(field, cam, lod=None) -> np.ndarray:
    """O1 + O4 for every Gaussian of ``field`` in one camera -> PROJ_DTYPE [n]
    (``lod``: optional synth.LodData, NEXT-2 opacity blending)."""
    L = lib()
    planes = np.ascontiguousarray(field.planes, dtype=np.float32)
    c = _cam(cam)
    out = np.zeros(field.n, dtype=PROJ_DTYPE)
    ls, keep = _lod(lod)
    L.orc_project(_p(planes), field.n, field.sh_degree, _p(c), ctypes.byref(ls) if ls else None, _p(out))
    return out


def lod_blend(d, D, delta):
    """eq:lod_blend, clamped (App. A.4): max(0, min(1, 0.5 - (d - D) / (2 delta)))."""
    return float(lib().orc_lod_blend(float(d), float(D), float(delta)))


def lod_weight(d, level, lod):
    """Opacity multiplier of a level-``level`` Gaussian at camera distance d."""
    ls, keep = _lod(lod)
    return float(lib().orc_lod_weight(float(d), int(level), ctypes.byref(ls)))


def row_span(proj_one, ty: int, cam):
    """O1 step 15: tile-column span [x0, x1) of tile row ``ty`` of one
    projected Gaussian (x0 = x1 = 0 when empty)."""
    L = lib()
    p = np.ascontiguousarray(np.asarray(proj_one, dtype=PROJ_DTYPE).reshape(1))
    x0, x1 = ctypes.c_uint32(0), ctypes.c_uint32(0)
    L.orc_row_span(_p(p), int(ty), _wh(cam)[0], ctypes.byref(x0), ctypes.byref(x1))
    return int(x0.value), int(x1.value)


def tiles_of(proj_one, cam):
    """All (ty, tx) tiles of one projected Gaussian in emission order."""
    if int(proj_one["n_tiles"]) == 0:
        return []
    out = []
    for ty in range(int(proj_one["py0"]) >> 4, (int(proj_one["py1"]) >> 4) + 1):
        x0, x1 = row_span(proj_one, ty, cam)
        out.extend((ty, tx) for tx in range(x0, x1))
    return out


def emit_keys(proj, cam, view_in_batch: int = 0):
    """O2: unsorted duplicated keys of one view, emission order (g, ty, tx)."""
    L = lib()
    c = _cam(cam)
    k = L.orc_count_keys(_p(proj), len(proj))
    keys = np.zeros(max(k, 1), dtype=np.uint64)
    vals = np.zeros(max(k, 1), dtype=np.uint32)
    L.orc_emit_keys(_p(proj), len(proj), _p(c), view_in_batch, _p(keys), _p(vals))
    return keys[:k], vals[:k]


def sort_pairs(keys, vals):
    """O3: (key, value) lexicographic order (qsort); returns sorted copies."""
    L = lib()
    k = np.array(keys, dtype=np.uint64, copy=True)
    v = np.array(vals, dtype=np.uint32, copy=True)
    L.orc_sort_pairs(_p(k), _p(v), len(k))
    return k, v


def ranges(sorted_keys, n_tiles_total: int):
    """O3: [start, end) per (view, tile) prefix; empty tiles get [s, s)."""
    L = lib()
    sk = np.ascontiguousarray(sorted_keys, dtype=np.uint64)
    out = np.zeros((n_tiles_total, 2), dtype=np.uint32)
    L.orc_ranges(_p(sk), len(sk), n_tiles_total, _p(out))
    return out


def bin_sort_batch(projs, cams):
    """O2 + O3 over a batch of same-resolution views: the expected outputs of
    gsr_bin_sort (unsorted keys/vals, sorted keys/vals, ranges [V*tiles][2])."""
    gx, gy = grid(cams[0])
    ks, vs = [], []
    for v, (p, c) in enumerate(zip(projs, cams)):
        k, val = emit_keys(p, c, v)
        ks.append(k)
        vs.append(val)
    keys = np.concatenate(ks) if ks else np.zeros(0, np.uint64)
    vals = np.concatenate(vs) if vs else np.zeros(0, np.uint32)
    sk, sv = sort_pairs(keys, vals)
    rg = ranges(sk, len(cams) * gx * gy)
    return dict(keys_unsorted=keys, vals_unsorted=vals, keys=sk, vals=sv, ranges=rg)


def composite_tiled(proj, sorted_vals, ranges_view, cam):
    """O5 + O6 tiled compositing of one view; ranges_view is that view's
    [tiles][2] slice with starts relative to ``sorted_vals``."""
    L = lib()
    c = _cam(cam)
    W, H = _wh(c)
    rgbu = np.zeros((H, W, 4), dtype=np.float32)
    tf = np.zeros((H, W), dtype=np.float32)
    nc = np.zeros((H, W), dtype=np.uint32)
    nf = np.zeros(2, dtype=np.uint64)
    sv = np.ascontiguousarray(sorted_vals, dtype=np.uint32)
    rv = np.ascontiguousarray(ranges_view, dtype=np.uint32)
    score = L.orc_composite_tiled(_p(proj), _p(sv if len(sv) else np.zeros(1, np.uint32)), _p(rv),
                                  _p(c), _p(rgbu), _p(tf), _p(nc), _p(nf))
    return dict(rgbu=rgbu, t_final=tf, n_contrib=nc, score=score, n_frag=int(nf[0]), n_eval=int(nf[1]))


def composite_trace(proj, sorted_vals, ranges_view, cam):
    """NEXT-3: per pixel (row-major), the Gaussians the O5 loop blends, in
    order -> (offsets int64 [H*W+1], idx uint32 [total])."""
    L = lib()
    c = _cam(cam)
    W, H = _wh(c)
    off = np.zeros(W * H + 1, dtype=np.int64)
    sv = np.ascontiguousarray(sorted_vals, dtype=np.uint32)
    rv = np.ascontiguousarray(ranges_view, dtype=np.uint32)
    svp = _p(sv if len(sv) else np.zeros(1, np.uint32))
    k = L.orc_composite_trace(_p(proj), svp, _p(rv), _p(c), _p(off), None, 0)
    idx = np.zeros(max(k, 1), dtype=np.uint32)
    L.orc_composite_trace(_p(proj), svp, _p(rv), _p(c), _p(off), _p(idx), k)
    return off, idx[:k]


def composite_brute(proj, cam):
    """O5 + O6 brute force: every pixel over all non-culled Gaussians in
    (depth bits, index) order, no tiles (tiny inputs)."""
    L = lib()
    c = _cam(cam)
    W, H = _wh(c)
    rgbu = np.zeros((H, W, 4), dtype=np.float32)
    tf = np.zeros((H, W), dtype=np.float32)
    nc = np.zeros((H, W), dtype=np.uint32)
    nf = np.zeros(2, dtype=np.uint64)
    score = L.orc_composite_brute(_p(proj), len(proj), _p(c), _p(rgbu), _p(tf), _p(nc), _p(nf))
    return dict(rgbu=rgbu, t_final=tf, n_contrib=nc, score=score, n_frag=int(nf[0]), n_eval=int(nf[1]))


def render_view(field, cam, lod=None):
    """O1..O6 for one view through the tiled path; returns a dict with the
    projection, bin-sort outputs, images and score."""
    p = project(field, cam, lod)
    bs = bin_sort_batch([p], np.asarray([cam]))
    out = composite_tiled(p, bs["vals"], bs["ranges"], cam)
    out.update(proj=p, **bs)
    return out


def render_views(field, cams, n_threads: int = 0, images: bool = False, lod=None):
    """O1..O6 for many views, one view per host thread (bench cpu_baseline).
    Returns (scores float64 [V], n_frag uint64 [V], n_keys int64 [V], rgbu or None)."""
    L = lib()
    cams = np.ascontiguousarray(cams)
    V = len(cams)
    planes = np.ascontiguousarray(field.planes, dtype=np.float32)
    scores = np.zeros(V, dtype=np.float64)
    nf = np.zeros(V, dtype=np.uint64)
    nk = np.zeros(V, dtype=np.int64)
    rgbu = None
    if images:
        W, H = _wh(cams[0])
        assert all(_wh(c) == (W, H) for c in cams)
        rgbu = np.zeros((V, H, W, 4), dtype=np.float32)
    if n_threads <= 0:
        n_threads = os.cpu_count() or 1
    ls, keep = _lod(lod)
    L.orc_render_views(_p(planes), field.n, field.sh_degree, _p(cams), V, ctypes.byref(ls) if ls else None,
                       n_threads, _p(rgbu), _p(scores), _p(nf), _p(nk))
    return scores, nf, nk, rgbu


def select_topk(scores, k: int, exclude=None):
    """O7 ("top-k poses by u(θ)"; App. A.2):
    order by (score descending, index ascending), drop excluded indices, take
    the first k.  k < 1 or k > #available raises ValueError (budget error)."""
    n = len(scores)
    ex = np.zeros(n, dtype=bool) if exclude is None else np.asarray(exclude, dtype=bool)
    avail = [i for i in range(n) if not ex[i]]
    if k < 1 or k > len(avail):
        raise ValueError("budget error: k must be in [1, #available]")
    order = sorted(avail, key=lambda i: (-float(scores[i]), i))
    return np.array(order[:k], dtype=np.int32)
