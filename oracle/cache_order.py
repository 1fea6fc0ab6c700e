"""NEXT-2b oracle: uncertainty-guided cached view-direction orderings
(§3.5: "multiple view-dependent Gaussian orderings are
pre-sorted and cached per tile ... tiles with mean uncertainty above a
threshold tau retain a larger set of cached orderings") -- TEST
INFRASTRUCTURE ONLY (same rules as the package docstring of oracle/).

Readings (SPEC lod-cache S:L571-591, design decisions S:L596-601):
  * a "tile" is a contiguous index range of the field (one placed Wang tile);
  * bins are azimuthal: b_k = (cos(2 pi k / B), 0, sin(2 pi k / B)), computed in
    float64 and rounded once to float32; B = 16 if the tile's mean
    uncertainty exceeds tau (= 0.6, §3.6 "tau=0.6"), else 8;
  * the ordering of bin k is the tile's Gaussians by ascending
    key = fl32(fl32(x bx) + fl32(z bz)) (front to back when looking along
    b_k), ties by index;
  * a view picks, per tile, the bin maximising <h, b_k> with h the horizontal
    part of its forward direction (float64, ties to the lower k), and visits
    the tiles front to back by <centre - eye, forward> (float64, ties to the
    lower tile);
  * the view's blend order is the concatenation; keys are emitted in it and
    every tile list is composited in it (the exact depth sort is skipped).
Pins: tests/test_oracle_cache_order.py.
"""
from __future__ import annotations

import math

import numpy as np

from . import _cam, _p, composite_tiled, grid, lib, project, ranges, sort_pairs

TAU = 0.6
BASE_BINS, HOT_BINS = 8, 16


def tile_mean_uncertainty(field, tile_start) -> np.ndarray:
    """Mean per-Gaussian uncertainty of each tile (the cache policy input)."""
    u = field.planes[1, :, 3].astype(np.float64)
    return np.array([u[tile_start[t]:tile_start[t + 1]].mean() for t in range(len(tile_start) - 1)])


def bins_for(u_bar, tau: float = TAU):
    """Cache policy: hot tiles (mean uncertainty > tau) keep 16 bins, else 8."""
    return HOT_BINS if float(u_bar) > tau else BASE_BINS


def bin_dirs(B: int) -> np.ndarray:
    """float32 [B][2] (bx, bz) of the azimuthal bin directions."""
    a = 2.0 * np.pi * np.arange(B) / B
    return np.stack([np.cos(a), np.sin(a)], 1).astype(np.float32)


def cached_orders(field, tile_start, B: int, t: int) -> np.ndarray:
    """[B][n_t] orderings (global Gaussian indices) of tile t."""
    s, e = int(tile_start[t]), int(tile_start[t + 1])
    x = field.planes[0, s:e, 0].astype(np.float32)
    z = field.planes[0, s:e, 2].astype(np.float32)
    out = np.zeros((B, e - s), dtype=np.uint32)
    for k, (bx, bz) in enumerate(bin_dirs(B)):
        key = (x * bx) + (z * bz)  # float32 products and sum, one rounding each
        out[k] = s + np.lexsort((np.arange(e - s), key))
    return out


def view_choice(cam, centres, bins):
    """(tile visiting order, chosen bin per tile) of one camera."""
    R = np.asarray(cam["R"], dtype=np.float64).reshape(3, 3)
    f = R[2]
    eye = np.asarray(cam["campos"], dtype=np.float64)
    h = np.array([f[0], f[2]])
    h = h / max(np.linalg.norm(h), 1e-30)
    choice = []
    for B in bins:
        a = 2.0 * np.pi * np.arange(B) / B
        dots = h[0] * np.cos(a) + h[1] * np.sin(a)
        choice.append(int(np.argmax(dots)))
    depth = (np.asarray(centres, dtype=np.float64) - eye) @ f
    order = np.lexsort((np.arange(len(centres)), depth))
    return order, choice


def view_order(field, tile_start, bins, centres, cam, caches=None):
    """The view's blend order (global indices) under the cached orderings."""
    order, choice = view_choice(cam, centres, bins)
    parts = []
    for t in order:
        c = caches[t] if caches is not None else cached_orders(field, tile_start, bins[t], t)
        parts.append(c[choice[t]])
    return np.concatenate(parts).astype(np.uint32)


def render_view_cached(field, cam, tile_start, bins, centres, lod=None, caches=None):
    """O1..O6 of one view with the cached blend order: keys emitted in it,
    (key, value) sort, tiled compositing."""
    L = lib()
    p = project(field, cam, lod)
    order = view_order(field, tile_start, bins, centres, cam, caches)
    c = _cam(cam)
    k = int(p["n_tiles"].astype(np.int64).sum())
    keys = np.zeros(max(k, 1), dtype=np.uint64)
    vals = np.zeros(max(k, 1), dtype=np.uint32)
    L.orc_emit_keys_order(_p(p), _p(order), len(order), _p(c), 0, _p(keys), _p(vals))
    sk, sv = sort_pairs(keys[:k], vals[:k])
    gx, gy = grid(cam)
    rg = ranges(sk, gx * gy)
    out = composite_tiled(p, sv, rg, cam)
    out.update(proj=p, vals=sv, ranges=rg, order=order)
    return out
