"""Thin ctypes binding of libgsr (include/gsr.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module
turns torch CUDA tensors / numpy camera arrays into the C-ABI's plain
pointers and raises ``GsrError`` on a non-OK status.  There is no CPU
fallback: if ``libgsr.so`` is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GSR_LIB") or os.path.join(_HERE, "libgsr.so")

GSR_OK, GSR_EINVAL, GSR_ECUDA, GSR_ENOMEM, GSR_ECAPACITY, GSR_EBUDGET = range(6)
STATUS_NAMES = {0: "GSR_OK", 1: "GSR_EINVAL", 2: "GSR_ECUDA", 3: "GSR_ENOMEM", 4: "GSR_ECAPACITY",
                5: "GSR_EBUDGET"}
GSR_MAX_VIEWS = 64
GSR_TILE = 16

# gsr_camera (96 bytes), field for field
CAM_DTYPE = np.dtype(
    [("R", "<f4", (9,)), ("t", "<f4", (3,)), ("campos", "<f4", (3,)), ("fx", "<f4"), ("fy", "<f4"),
     ("cx", "<f4"), ("cy", "<f4"), ("limx", "<f4"), ("limy", "<f4"), ("znear", "<f4"),
     ("width", "<i4"), ("height", "<i4")], align=True)
assert CAM_DTYPE.itemsize == 96

EXPORTED = ["gsr_create", "gsr_destroy", "gsr_last_error", "gsr_version", "gsr_camera_look_at",
            "gsr_project", "gsr_bin_sort", "gsr_composite", "gsr_score_views", "gsr_select_nbv",
            "gsr_sort_pairs_u64", "gsr_scratch_bytes", "gsr_timing_enable", "gsr_timing_read", "gsr_w2_scores",
            "gsr_sobel_scores", "gsr_backward", "gsr_order_cache_size", "gsr_build_order_cache",
            "gsr_bin_sort_cached", "gsr_l2_loss", "gsr_adam_step", "gsr_order_cache_bins",
            "gsr_set_composite_residency", "gsr_upload", "gsr_download"]
STAGES = ["project", "compact", "depth_sort", "emit", "ranges", "tile_sort", "composite", "score", "select",
          "sort_u64", "w2", "sobel", "backward", "optim", "backward_project"]


class GsrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Gaussians(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_degree", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("pos_opacity", ctypes.c_void_p), ("scale_unc", ctypes.c_void_p), ("rot", ctypes.c_void_p),
                ("sh", ctypes.c_void_p)]


class _Lod(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("delta", ctypes.c_float), ("thresholds", ctypes.c_float * 7),
                ("tile_level", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libgsr.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, i64, i32, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
    L.gsr_create.argtypes = [ctypes.POINTER(P), ctypes.c_int]
    L.gsr_destroy.argtypes = [P]
    L.gsr_last_error.argtypes = [P]
    L.gsr_last_error.restype = ctypes.c_char_p
    L.gsr_version.restype = ctypes.c_char_p
    L.gsr_camera_look_at.argtypes = [ctypes.c_double] * 3 + [P, i32, i32, ctypes.c_double, ctypes.c_double, P]
    L.gsr_project.argtypes = [P, P, P, i32, P, P, P, P]
    L.gsr_bin_sort.argtypes = [P, P, i64, P, i32, P, P, i64, P, P, P, P, P]
    L.gsr_composite.argtypes = [P, P, i64, P, P, P, i32, P, P, P, P, P, P, P]
    L.gsr_sobel_scores.argtypes = [P, P, P, i32, P, P, P]
    L.gsr_backward.argtypes = [P, P, P, i32, P, P, P, P, P, P, P, P, P]
    L.gsr_l2_loss.argtypes = [P, P, P, i64, P, P, P, P]
    L.gsr_adam_step.argtypes = [P, P, P, P, P, i64, i32, P, ctypes.c_float, ctypes.c_float, ctypes.c_float, i32, P]
    L.gsr_order_cache_bins.argtypes = [P, P, P, i32, ctypes.c_float, i32, i32, P, P]
    L.gsr_order_cache_size.argtypes = [P, i32, P]
    L.gsr_order_cache_size.restype = i64
    L.gsr_build_order_cache.argtypes = [P, P, P, i32, P, P, P]
    L.gsr_bin_sort_cached.argtypes = [P, P, i64, P, i32, P, P, i32, P, P, P, P, i64, P, P, P]
    L.gsr_score_views.argtypes = [P, P, P, i32, P, P]
    L.gsr_select_nbv.argtypes = [P, P, i32, P, i32, P, P]
    L.gsr_sort_pairs_u64.argtypes = [P, P, P, P, P, i64, i32, i32, P]
    L.gsr_w2_scores.argtypes = [P, P, P, i32, i32, i32, i64, P, P, P]
    L.gsr_timing_enable.argtypes = [P, ctypes.c_int]
    L.gsr_set_composite_residency.argtypes = [P, i32]
    L.gsr_timing_read.argtypes = [P, P, P, P]
    L.gsr_scratch_bytes.argtypes = [P]
    L.gsr_upload.argtypes = [P, P, P, i64, P]
    L.gsr_download.argtypes = [P, P, P, i64, P]
    L.gsr_scratch_bytes.restype = i64
    for name in EXPORTED:
        if name not in ("gsr_last_error", "gsr_version", "gsr_scratch_bytes", "gsr_order_cache_size"):
            getattr(L, name).restype = st
    return L


lib = _load()


def version() -> str:
    return lib.gsr_version().decode()


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def cams_array(cams) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(cams).reshape(-1))
    if a.dtype != CAM_DTYPE:
        a = a.astype(CAM_DTYPE)
    return a


def gsr_camera_look_at(elevation: float, azimuth: float, radius: float, target, width: int, height: int,
                       focal: float, znear: float = 0.2) -> np.ndarray:
    """H1: θ = (elevation, azimuth, radius) -> one camera struct."""
    out = np.zeros(1, dtype=CAM_DTYPE)
    tgt = np.ascontiguousarray(np.asarray(target, dtype=np.float64).reshape(3))
    st = lib.gsr_camera_look_at(elevation, azimuth, radius, tgt.ctypes.data, width, height, focal, znear,
                                out.ctypes.data)
    if st != GSR_OK:
        raise GsrError(st, lib.gsr_last_error(None).decode())
    return out[0]


class Gaussians:
    """Device-resident packed field: planes[P][n][4] float32 CUDA tensor."""

    def __init__(self, planes, sh_degree: int):
        # the kernels read float4 planes: any other dtype would be misread silently
        if not planes.is_cuda or planes.dtype != torch.float32 or planes.dim() != 3 or planes.shape[-1] != 4:
            raise ValueError("Gaussians: planes must be a CUDA float32 tensor [P][n][4]")
        sh_degree = int(sh_degree)
        if not 0 <= sh_degree <= 3:
            raise ValueError("Gaussians: sh_degree must be in [0, 3]")
        need = 3 + (3 * (sh_degree + 1) ** 2 + 3) // 4  # (x,y,z,o), (s,u), q, SH slots
        if planes.shape[1] > 0 and planes.shape[0] < need:  # an empty field reads no plane
            raise ValueError(f"Gaussians: {planes.shape[0]} planes, degree {sh_degree} needs {need}")
        self.planes = planes.contiguous()
        self.sh_degree = sh_degree
        self.n = int(planes.shape[1])

    def struct(self) -> _Gaussians:
        base = self.planes.data_ptr()
        stride = self.n * 16
        return _Gaussians(self.n, self.sh_degree, 0, base, base + stride, base + 2 * stride, base + 3 * stride)


class Lod:
    """NEXT-2 LOD blending (gsr_lod): device tile_level [n][4] float32 tensor
    (tile centre x, y, z, level) + levels, bandwidth delta and thresholds."""

    def __init__(self, tile_level, levels: int, delta: float, thresholds):
        if not tile_level.is_cuda or tile_level.dtype != torch.float32 or tile_level.shape[-1] != 4:
            raise ValueError("Lod: tile_level must be a CUDA float32 tensor [n][4]")
        self.tile_level = tile_level.contiguous()
        self.levels = int(levels)
        self.delta = float(delta)
        self.thresholds = [float(x) for x in thresholds]

    def struct(self) -> _Lod:
        th = (ctypes.c_float * 7)(*(self.thresholds + [0.0] * (7 - len(self.thresholds))))
        return _Lod(self.levels, self.delta, th, self.tile_level.data_ptr())


class Context:
    """A gsr_ctx (scratch owner) bound to one device; one per stream/thread."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        st = lib.gsr_create(ctypes.byref(h), device)
        if st != GSR_OK:
            raise GsrError(st, lib.gsr_last_error(None).decode())
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            lib.gsr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != GSR_OK:
            raise GsrError(st, lib.gsr_last_error(self.handle).decode())

    def scratch_bytes(self) -> int:
        return int(lib.gsr_scratch_bytes(self.handle))

    def set_composite_residency(self, blocks_per_sm: int):
        """K6 launch shape: 0 = one block per strip; k > 0 = persistent grid of
        k blocks per SM (leaves room for kernels on other streams)."""
        self._check(lib.gsr_set_composite_residency(self.handle, int(blocks_per_sm)))

    def timing(self, enable: bool = True):
        self._check(lib.gsr_timing_enable(self.handle, 1 if enable else 0))

    def timing_read(self) -> dict:
        """SYNC: per-stage {ms, launches, bytes} since the last read (then reset)."""
        ms = np.zeros(len(STAGES), np.float64)
        la = np.zeros(len(STAGES), np.int64)
        by = np.zeros(len(STAGES), np.float64)
        self._check(lib.gsr_timing_read(self.handle, ms.ctypes.data, la.ctypes.data, by.ctypes.data))
        return {s: dict(ms=float(ms[i]), launches=int(la[i]), bytes=float(by[i])) for i, s in enumerate(STAGES)}


def gsr_project(ctx: Context, g: Gaussians, cams, render_rec, bin_rec, stream=None, lod: Optional[Lod] = None):
    c = cams_array(cams)
    gs = g.struct()
    ls = lod.struct() if lod is not None else None
    ctx._check(lib.gsr_project(ctx.handle, ctypes.byref(gs), c.ctypes.data, len(c),
                               ctypes.byref(ls) if ls is not None else None, _ptr(render_rec), _ptr(bin_rec),
                               _stream(stream)))


def gsr_bin_sort(ctx: Context, bin_rec, n: int, cams, vals, capacity: int, ranges, keys=None,
                 keys_unsorted=None, vals_unsorted=None, stream=None) -> int:
    """Returns K (SYNC readback).  Raises GsrError(GSR_ECAPACITY) with .required = K."""
    c = cams_array(cams)
    nk = ctypes.c_int64(0)
    st = lib.gsr_bin_sort(ctx.handle, _ptr(bin_rec), n, c.ctypes.data, len(c), _ptr(keys), _ptr(vals), capacity,
                          ctypes.byref(nk), _ptr(ranges), _ptr(keys_unsorted), _ptr(vals_unsorted),
                          _stream(stream))
    if st == GSR_ECAPACITY:
        e = GsrError(st, lib.gsr_last_error(ctx.handle).decode())
        e.required = int(nk.value)
        raise e
    ctx._check(st)
    return int(nk.value)


class OrderCache:
    """NEXT-2b: the field's cached view-direction orderings (device) + the
    tile table (host): tile_start int64 [n_tiles + 1], bins int32 [n_tiles],
    centres float64 [n_tiles][3]."""

    def __init__(self, ctx: "Context", g: Gaussians, tile_start, bins, centres, stream=None):
        import torch
        self.tile_start = np.ascontiguousarray(np.asarray(tile_start, dtype=np.int64))
        self.bins = np.ascontiguousarray(np.asarray(bins, dtype=np.int32))
        self.centres = np.ascontiguousarray(np.asarray(centres, dtype=np.float64).reshape(-1, 3))
        self.n_tiles = len(self.bins)
        size = int(lib.gsr_order_cache_size(self.tile_start.ctypes.data, self.n_tiles, self.bins.ctypes.data))
        self.cache = torch.empty(max(size, 1), dtype=torch.int32, device=g.planes.device)
        gs = g.struct()
        ctx._check(lib.gsr_build_order_cache(ctx.handle, ctypes.byref(gs), self.tile_start.ctypes.data,
                                             self.n_tiles, self.bins.ctypes.data, _ptr(self.cache),
                                             _stream(stream)))


def gsr_bin_sort_cached(ctx: Context, bin_rec, n: int, cams, oc: OrderCache, vals, capacity: int, ranges,
                        keys=None, stream=None) -> int:
    """gsr_bin_sort with the cached blend order (NEXT-2b); returns K."""
    c = cams_array(cams)
    nk = ctypes.c_int64(0)
    st = lib.gsr_bin_sort_cached(ctx.handle, _ptr(bin_rec), n, c.ctypes.data, len(c), _ptr(oc.cache),
                                 oc.tile_start.ctypes.data, oc.n_tiles, oc.bins.ctypes.data, oc.centres.ctypes.data,
                                 _ptr(keys), _ptr(vals), capacity, ctypes.byref(nk), _ptr(ranges), _stream(stream))
    if st == GSR_ECAPACITY:
        e = GsrError(st, lib.gsr_last_error(ctx.handle).decode())
        e.required = int(nk.value)
        raise e
    ctx._check(st)
    return int(nk.value)


def gsr_order_cache_bins(ctx: Context, g: Gaussians, tile_start, tau: float, base_bins: int = 8,
                         hot_bins: int = 16, stream=None) -> np.ndarray:
    """NEXT-2b cache policy (§3.5, tau §3.6): bins per
    tile from the tiles' mean uncertainty (computed in libgsr; SYNC)."""
    start = np.ascontiguousarray(np.asarray(tile_start, dtype=np.int64))
    bins = np.zeros(len(start) - 1, dtype=np.int32)
    ctx._check(lib.gsr_order_cache_bins(ctx.handle, ctypes.byref(g.struct()), start.ctypes.data, len(bins),
                                        float(tau), int(base_bins), int(hot_bins), bins.ctypes.data,
                                        _stream(stream)))
    return bins


def gsr_composite(ctx: Context, render_rec, n: int, vals, ranges, cams, tile_partial, rgbu=None, t_final=None,
                  n_contrib=None, n_frag=None, gray=None, stream=None):
    c = cams_array(cams)
    ctx._check(lib.gsr_composite(ctx.handle, _ptr(render_rec), n, _ptr(vals), _ptr(ranges), c.ctypes.data, len(c),
                                 _ptr(rgbu), _ptr(t_final), _ptr(n_contrib), _ptr(gray), _ptr(tile_partial),
                                 _ptr(n_frag), _stream(stream)))


def gsr_backward(ctx: Context, g: Gaussians, cams, render_rec, bin_rec, vals, ranges, rgbu, dl_drgbu, grads,
                 lod: Optional["Lod"] = None, stream=None):
    """NEXT-3: ADD dL/dparams ([P][n][4], the field's plane layout) for the
    upstream image gradient dl_drgbu [V][H][W][4] of this batch's forward."""
    c = cams_array(cams)
    gs = g.struct()
    ls = lod.struct() if lod is not None else None
    ctx._check(lib.gsr_backward(ctx.handle, ctypes.byref(gs), c.ctypes.data, len(c),
                                ctypes.byref(ls) if ls is not None else None, _ptr(render_rec), _ptr(bin_rec),
                                _ptr(vals), _ptr(ranges), _ptr(rgbu), _ptr(dl_drgbu), _ptr(grads), _stream(stream)))


def gsr_l2_loss(ctx: Context, img, target, weights, dl_dimg=None, loss=None, stream=None):
    """NEXT-3: L2 photometric loss over (r, g, b, U) pixels (+ its gradient)."""
    import torch
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float32).reshape(4))
    if loss is None:
        loss = torch.zeros(1, dtype=torch.float64, device=img.device)
    ctx._check(lib.gsr_l2_loss(ctx.handle, _ptr(img), _ptr(target), int(img.numel() // 4), w.ctypes.data,
                               _ptr(dl_dimg), _ptr(loss), _stream(stream)))
    return loss


def gsr_adam_step(ctx: Context, params, grads, m, v, lr, step: int, beta1=0.9, beta2=0.999, eps=1e-8,
                  stream=None):
    """NEXT-3: projected Adam on the field planes [P][n][4] (lr [P][4] host)."""
    P, n = int(params.shape[0]), int(params.shape[1])
    lr = np.ascontiguousarray(np.asarray(lr, dtype=np.float32).reshape(P, 4))
    ctx._check(lib.gsr_adam_step(ctx.handle, _ptr(params), _ptr(grads), _ptr(m), _ptr(v), n, P, lr.ctypes.data,
                                 beta1, beta2, eps, step, _stream(stream)))


def gsr_sobel_scores(ctx: Context, gray, cams, tile_partial, scores, stream=None):
    """NEXT-4 (PAPER.md eq:uncert_img): mean Sobel gradient magnitude of gray [V][H][W]."""
    c = cams_array(cams)
    ctx._check(lib.gsr_sobel_scores(ctx.handle, _ptr(gray), c.ctypes.data, len(c), _ptr(tile_partial), _ptr(scores),
                                    _stream(stream)))


def gsr_score_views(ctx: Context, tile_partial, cams, scores, stream=None):
    c = cams_array(cams)
    ctx._check(lib.gsr_score_views(ctx.handle, _ptr(tile_partial), c.ctypes.data, len(c), _ptr(scores),
                                   _stream(stream)))


def gsr_upload(ctx: Context, dst, src, stream=None):
    """Host -> device copy of ``src`` (host tensor / ndarray; page-locked for
    an asynchronous copy) into the CUDA tensor ``dst`` on ``stream``."""
    nb = _nbytes(src)
    if nb != _nbytes(dst):
        raise ValueError("gsr_upload: size mismatch")
    ctx._check(lib.gsr_upload(ctx.handle, _ptr(dst), _ptr(src), nb, _stream(stream)))


def gsr_download(ctx: Context, dst, src, stream=None):
    """Device -> host copy of the CUDA tensor ``src`` into the host tensor /
    ndarray ``dst`` on ``stream`` (valid once the stream has synchronised)."""
    nb = _nbytes(src)
    if nb != _nbytes(dst):
        raise ValueError("gsr_download: size mismatch")
    ctx._check(lib.gsr_download(ctx.handle, _ptr(dst), _ptr(src), nb, _stream(stream)))


def _nbytes(t) -> int:
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("host staging needs a contiguous array")
        return int(t.nbytes)
    if not t.is_contiguous():
        raise ValueError("host staging needs a contiguous tensor")
    return int(t.numel() * t.element_size())


def gsr_select_nbv(ctx: Context, scores, k: int, out_idx, exclude: Optional[np.ndarray] = None, stream=None):
    ex = None if exclude is None else np.ascontiguousarray(np.asarray(exclude, dtype=np.uint8))
    ctx._check(lib.gsr_select_nbv(ctx.handle, _ptr(scores), int(scores.numel()), _ptr(ex), k, _ptr(out_idx),
                                  _stream(stream)))


def gsr_sort_pairs_u64(ctx: Context, keys_in, vals_in, keys_out, vals_out, begin_bit: int = 0, end_bit: int = 64,
                       stream=None):
    ctx._check(lib.gsr_sort_pairs_u64(ctx.handle, _ptr(keys_in), _ptr(vals_in), _ptr(keys_out), _ptr(vals_out),
                                      int(keys_in.numel()), begin_bit, end_bit, _stream(stream)))


def gsr_w2_scores(ctx: Context, mu, s2, scores, map_out=None, stream=None):
    """NEXT-1 (PAPER.md eq:w2_pixel): mu, s2 CUDA float tensors [V][M][C][HW]."""
    V, M, C, HW = (int(x) for x in mu.shape)
    assert tuple(s2.shape) == (V, M, C, HW) and mu.is_contiguous() and s2.is_contiguous()
    ctx._check(lib.gsr_w2_scores(ctx.handle, _ptr(mu), _ptr(s2), V, M, C, HW, _ptr(scores), _ptr(map_out),
                                 _stream(stream)))
