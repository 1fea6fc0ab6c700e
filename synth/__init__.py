"""Seeded synthetic inputs shared by the CUDA path, the oracle and the bench.

This module holds NO arithmetic of the method (no projection, no sorting, no
compositing, no scoring).  It only draws Gaussian fields and builds camera
structs, exactly as BASELINE.json ``configs`` and SURVEY.md §8(d) describe:

* Gaussian draws (SURVEY §8(d) "Generator rules"): numpy ``Generator(PCG64(seed))``;
  draw order means, log-scales (N×3), quaternions (N×4 N(0,1)), opacity logits,
  SH (DC N×3, then rest N×15×3), uncertainty.  Activations (exp of log-scales,
  sigmoid of logits, quaternion normalisation) are done in float64 and rounded
  once to float32 (SURVEY §8(c) reading "Stored activations").
* Cameras: the θ = (elevation, azimuth, radius) triple of PAPER.md L57
  (§3.1 Problem definition), placed on a Fibonacci hemisphere,
  looking at the origin.  Look-at frame, OpenCV axes (x right, y down,
  z forward), world up +y (SURVEY §8(c) reading "Camera model").  Built in
  float64, rounded once to float32.

The packed field layout is the one the C-ABI (include/gsr.h) takes:
``planes[P][n][4]`` float32, plane 0 = (x, y, z, opacity), plane 1 =
(sx, sy, sz, uncertainty), plane 2 = (qw, qx, qy, qz), planes 3.. = SH
coefficients slot-major (plane 3+j, element i holds flat coefficients
4j..4j+3 of Gaussian i, flat index = 3*coef + channel).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field
from typing import Optional

import numpy as np

# --------------------------------------------------------------------------
# camera struct (mirrors gsr_camera in include/gsr.h; 96 bytes)
# --------------------------------------------------------------------------
CAM_DTYPE = np.dtype(
    [
        ("R", "<f4", (9,)),
        ("t", "<f4", (3,)),
        ("campos", "<f4", (3,)),
        ("fx", "<f4"),
        ("fy", "<f4"),
        ("cx", "<f4"),
        ("cy", "<f4"),
        ("limx", "<f4"),
        ("limy", "<f4"),
        ("znear", "<f4"),
        ("width", "<i4"),
        ("height", "<i4"),
    ],
    align=True,
)
assert CAM_DTYPE.itemsize == 96

ZNEAR = 0.2  # BASELINE.json configs[0] "near plane 0.2" (used for every config)


def n_sh_planes(sh_degree: int) -> int:
    """ceil(3 (d+1)^2 / 4) float4 planes hold the SH coefficients."""
    return (3 * (sh_degree + 1) ** 2 + 3) // 4


def look_at(eye, target, width: int, height: int, focal: float, znear: float = ZNEAR):
    """One camera struct (float64 maths, rounded once to float32).

    f = normalize(target - eye); r = normalize(f x up); d = f x r; rows of R
    are (r, d, f); t = -R eye; up = +y unless |f.y| > 0.9999, then +z.
    Principal point (W/2, H/2); limx = 1.3 (W/2)/fx, limy = 1.3 (H/2)/fy.
    """
    eye = np.asarray(eye, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    f = target - eye
    f = f / np.linalg.norm(f)
    up = np.array([0.0, 1.0, 0.0])
    if abs(f[1]) > 0.9999:
        up = np.array([0.0, 0.0, 1.0])
    r = np.cross(f, up)
    r = r / np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f])
    t = -R @ eye
    cam = np.zeros((), dtype=CAM_DTYPE)
    cam["R"] = R.reshape(-1).astype(np.float32)
    cam["t"] = t.astype(np.float32)
    cam["campos"] = eye.astype(np.float32)
    cam["fx"] = np.float32(focal)
    cam["fy"] = np.float32(focal)
    cam["cx"] = np.float32(width / 2.0)
    cam["cy"] = np.float32(height / 2.0)
    cam["limx"] = np.float32(1.3 * (width / 2.0) / focal)
    cam["limy"] = np.float32(1.3 * (height / 2.0) / focal)
    cam["znear"] = np.float32(znear)
    cam["width"] = width
    cam["height"] = height
    return cam


def camera_from_theta(elev: float, azim: float, radius: float, width: int, height: int,
                      focal: float, target=(0.0, 0.0, 0.0), znear: float = ZNEAR):
    """θ = (elevation, azimuth, radius) of PAPER.md L57 → camera struct.

    eye = target + radius (cos e cos a, sin e, cos e sin a)  (world up +y).
    """
    eye = np.asarray(target, dtype=np.float64) + radius * np.array(
        [math.cos(elev) * math.cos(azim), math.sin(elev), math.cos(elev) * math.sin(azim)])
    return look_at(eye, target, width, height, focal, znear)


def fibonacci_eyes(n: int, radius: float, y_min: float = 0.0, y_max: float = 1.0) -> np.ndarray:
    """y_i = y_max - (i+1/2)(y_max-y_min)/n; rho = sqrt(1-y^2);
    phi_i = i pi (3 - sqrt 5); eye = R (rho cos phi, y, rho sin phi)."""
    i = np.arange(n, dtype=np.float64)
    y = y_max - (i + 0.5) * (y_max - y_min) / n
    rho = np.sqrt(1.0 - y * y)
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    return radius * np.stack([rho * np.cos(phi), y, rho * np.sin(phi)], axis=1)


def fibonacci_cameras(n: int, radius: float, width: int, height: int, focal: float,
                      y_min: float = 0.0, y_max: float = 1.0) -> np.ndarray:
    eyes = fibonacci_eyes(n, radius, y_min, y_max)
    cams = np.zeros(n, dtype=CAM_DTYPE)
    for k in range(n):
        cams[k] = look_at(eyes[k], (0.0, 0.0, 0.0), width, height, focal)
    return cams


def flyover_cameras(n: int, width: int, height: int, focal: float) -> np.ndarray:
    """Config 4 path (SURVEY §8(c) reading "Config 4 details"):
    eye_i = (2 + cos phi_i, 1.5, 2 + sin phi_i), phi_i = 2 pi i / n,
    yaw = phi_i + 90 deg, pitch = -30 deg."""
    cams = np.zeros(n, dtype=CAM_DTYPE)
    pitch = math.radians(-30.0)
    for i in range(n):
        phi = 2.0 * math.pi * i / n
        eye = np.array([2.0 + math.cos(phi), 1.5, 2.0 + math.sin(phi)])
        yaw = phi + math.pi / 2.0
        fwd = np.array([math.cos(pitch) * math.cos(yaw), math.sin(pitch),
                        math.cos(pitch) * math.sin(yaw)])
        cams[i] = look_at(eye, eye + fwd, width, height, focal)
    return cams


def with_resolution(cams: np.ndarray, width: int, height: int, focal: float) -> np.ndarray:
    """Same poses, new image size / focal (config 5 fine pass)."""
    out = cams.copy()
    for c in out:
        c["fx"] = np.float32(focal)
        c["fy"] = np.float32(focal)
        c["cx"] = np.float32(width / 2.0)
        c["cy"] = np.float32(height / 2.0)
        c["limx"] = np.float32(1.3 * (width / 2.0) / focal)
        c["limy"] = np.float32(1.3 * (height / 2.0) / focal)
        c["width"] = width
        c["height"] = height
    return out


# --------------------------------------------------------------------------
# Gaussian field
# --------------------------------------------------------------------------
@dataclass
class GaussianField:
    planes: np.ndarray  # float32 [P][n][4], C-contiguous
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.planes.shape[1])

    @property
    def pos_opacity(self):
        return self.planes[0]

    @property
    def scale_unc(self):
        return self.planes[1]

    @property
    def rot(self):
        return self.planes[2]

    @property
    def sh(self):
        return self.planes[3:]

    def subset(self, idx) -> "GaussianField":
        return GaussianField(np.ascontiguousarray(self.planes[:, idx, :]), self.sh_degree)


def pack_field(means, scales, quats, opac, sh, unc, sh_degree: int) -> GaussianField:
    """Pack float64 activated arrays into float32 planes (one rounding)."""
    n = means.shape[0]
    ncoef = (sh_degree + 1) ** 2
    P = 3 + n_sh_planes(sh_degree)
    planes = np.zeros((P, n, 4), dtype=np.float32)
    planes[0, :, 0:3] = means
    planes[0, :, 3] = opac
    planes[1, :, 0:3] = scales
    planes[1, :, 3] = unc
    planes[2] = quats
    flat = np.zeros((n, 4 * n_sh_planes(sh_degree)), dtype=np.float64)
    flat[:, : 3 * ncoef] = np.asarray(sh, dtype=np.float64).reshape(n, 3 * ncoef)
    planes[3:] = flat.reshape(n, -1, 4).transpose(1, 0, 2).astype(np.float32)
    return GaussianField(np.ascontiguousarray(planes), sh_degree)


def _activate(rng, n, logscale_mu, logscale_sd, logit_mu, means):
    logs = rng.normal(logscale_mu, logscale_sd, size=(n, 3))
    q = rng.normal(0.0, 1.0, size=(n, 4))
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    logit = rng.normal(logit_mu, 1.0, size=n)
    return np.exp(logs), q, 1.0 / (1.0 + np.exp(-logit))


def gen_config1_field(n: int = 10_000, seed: int = 0) -> GaussianField:
    """configs[0]: mu ~ U[-1,1]^3; log s ~ N(-4,0.5); o = sigmoid(N(0,1));
    deg-0 RGB ~ U[0,1]; u ~ U[0,1]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    means = rng.uniform(-1.0, 1.0, size=(n, 3))
    scales, q, opac = _activate(rng, n, -4.0, 0.5, 0.0, means)
    dc = rng.uniform(0.0, 1.0, size=(n, 3))
    unc = rng.uniform(0.0, 1.0, size=n)
    return pack_field(means, scales, q, opac, dc.reshape(n, 1, 3), unc, 0)


def gen_terrain_field(n: int, seed: int, lo: float, hi: float, sh_degree: int = 3,
                      offset=(0.0, 0.0, 0.0), logscale_mu: float = -4.5) -> GaussianField:
    """configs[1..4]: x,z ~ U[lo,hi]; y = 0.1 sin(3x) cos(3z) + N(0,0.02);
    log s ~ N(-4.5,0.6); o = sigmoid(N(0.5,1)); SH DC ~ U[0,1], rest N(0,0.05);
    u ~ Beta(2,5).  ``offset`` translates (config 4 tile placement)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    xz = rng.uniform(lo, hi, size=(n, 2))
    noise = rng.normal(0.0, 0.02, size=n)
    x, z = xz[:, 0], xz[:, 1]
    y = 0.1 * np.sin(3.0 * x) * np.cos(3.0 * z) + noise
    means = np.stack([x, y, z], axis=1) + np.asarray(offset, dtype=np.float64)
    scales, q, opac = _activate(rng, n, logscale_mu, 0.6, 0.5, means)
    ncoef = (sh_degree + 1) ** 2
    sh = np.zeros((n, ncoef, 3))
    sh[:, 0, :] = rng.uniform(0.0, 1.0, size=(n, 3))
    if ncoef > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, size=(n, ncoef - 1, 3))
    unc = rng.beta(2.0, 5.0, size=n)
    return pack_field(means, scales, q, opac, sh, unc, sh_degree)


def concat_fields(fields) -> GaussianField:
    deg = fields[0].sh_degree
    assert all(f.sh_degree == deg for f in fields)
    return GaussianField(np.ascontiguousarray(np.concatenate([f.planes for f in fields], axis=1)), deg)


# Wang-tile edge colours for config 4 (SURVEY §8(c) "Config 4 details"):
# tile t has N = t&1, W = (t>>1)&1, S = E = (t>>2)&1, so every (N, W) pair
# has exactly two tiles.
def wang_tile_edges(t: int):
    return {"N": t & 1, "W": (t >> 1) & 1, "S": (t >> 2) & 1, "E": (t >> 2) & 1}


def wang_assignment(grid: int = 4, seed: int = 0) -> np.ndarray:
    """Scanline, seeded uniform choice among edge-compatible tiles."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = np.full((grid, grid), -1, dtype=np.int64)  # a[j (row, z), i (col, x)]
    for j in range(grid):
        for i in range(grid):
            ok = []
            for t in range(8):
                e = wang_tile_edges(t)
                if i > 0 and e["W"] != wang_tile_edges(a[j, i - 1])["E"]:
                    continue
                if j > 0 and e["N"] != wang_tile_edges(a[j - 1, i])["S"]:
                    continue
                ok.append(t)
            a[j, i] = ok[int(rng.integers(len(ok)))]
    return a


def gen_config4_field(n_per_tile: int = 500_000) -> GaussianField:
    tiles = [None] * 8
    assign = wang_assignment()
    parts = []
    for j in range(4):
        for i in range(4):
            t = int(assign[j, i])
            # each distinct tile is the same draw (seed 1000+t) placed at (i, 0, j)
            parts.append(gen_terrain_field(n_per_tile, 1000 + t, 0.0, 1.0, 3, offset=(i, 0.0, j)))
    return concat_fields(parts)


# --------------------------------------------------------------------------
# NEXT-2 LOD data (§3.5 eq:lod_blend; tab:dav-gswt-lod L205-246)
# --------------------------------------------------------------------------
@dataclass
class LodData:
    """Per-Gaussian (tile centre x, y, z, level) + the blend parameters."""
    tile_level: np.ndarray  # float32 [n][4]
    levels: int
    delta: float
    thresholds: tuple


# Readings: six levels (§4.4), thresholds doubling from 1.5 tile
# widths, bandwidth 0.25 (2 delta < every threshold gap); each
# coarser level has 1/4 of the Gaussians (tab:dav-gswt-lod: 3.7-3.9x per level)
# and 2.3x the scale (0.0032 -> 0.20 over five levels in the same table).
LOD_LEVELS = 6
LOD_THRESHOLDS = (1.5, 3.0, 6.0, 12.0, 24.0)
LOD_DELTA = 0.25
LOD_COUNT_STEP = 4
LOD_SCALE_STEP = 2.3


def gen_lod_tile(n0: int, seed: int, offset=(0.0, 0.0, 0.0), levels: int = LOD_LEVELS):
    """One unit-square terrain tile with ``levels`` LOD levels drawn as in
    configs[1] (level l: n0 / 4^l Gaussians, log-scale mean -4.5 + l ln 2.3,
    seed 16 seed + l).  Returns (field, tile_level [n][4])."""
    parts, tl = [], []
    centre = (offset[0] + 0.5, offset[1], offset[2] + 0.5)
    for l in range(levels):
        nl = max(1, n0 // LOD_COUNT_STEP ** l)
        parts.append(gen_terrain_field(nl, 16 * seed + l, 0.0, 1.0, 3, offset,
                                       logscale_mu=-4.5 + l * math.log(LOD_SCALE_STEP)))
        t = np.zeros((nl, 4), dtype=np.float32)
        t[:, 0:3] = centre
        t[:, 3] = l
        tl.append(t)
    return concat_fields(parts), np.concatenate(tl)


def gen_config4_lod(n_per_tile: int = 500_000):
    """configs[3] with NEXT-2 LOD levels: the 4x4 Wang assembly of 8 distinct
    tiles, each tile carrying six levels; returns (field, LodData)."""
    assign = wang_assignment()
    fields, tls = [], []
    for j in range(4):
        for i in range(4):
            t = int(assign[j, i])
            f, tl = gen_lod_tile(n_per_tile, 1000 + t, offset=(i, 0.0, j))
            fields.append(f)
            tls.append(tl)
    return concat_fields(fields), LodData(np.ascontiguousarray(np.concatenate(tls)), LOD_LEVELS, LOD_DELTA,
                                          LOD_THRESHOLDS)


def config4_tiles(n_per_tile: int = 500_000, lod: bool = False):
    """NEXT-2b tile structure of configs[3]: (tile_start int64 [17], centres
    float64 [16][3]) of the 16 placed tiles in field order (row j, column i);
    with ``lod`` the six levels of a placement are contiguous."""
    per = sum(max(1, n_per_tile // LOD_COUNT_STEP ** l) for l in range(LOD_LEVELS)) if lod else n_per_tile
    start = np.arange(17, dtype=np.int64) * per
    centres = np.array([[i + 0.5, 0.0, j + 0.5] for j in range(4) for i in range(4)], dtype=np.float64)
    return start, centres


def random_lod(rng, n: int, levels: int = 4, thresholds=(1.0, 2.0, 3.0), delta: float = 0.3,
               centre_range: float = 1.5) -> LodData:
    """Random tile centres and levels for parity tests."""
    tl = np.zeros((n, 4), dtype=np.float32)
    tl[:, 0:3] = rng.uniform(-centre_range, centre_range, size=(n, 3))
    tl[:, 3] = rng.integers(0, levels, size=n)
    return LodData(tl, levels, delta, tuple(thresholds))


# --------------------------------------------------------------------------
# configs
# --------------------------------------------------------------------------
@dataclass
class Scene:
    name: str
    field: GaussianField
    cameras: np.ndarray
    fine_width: int = 0
    fine_focal: float = 0.0
    top_k: int = 1
    meta: dict = dc_field(default_factory=dict)


CONFIG_NAMES = {
    1: "c1-tiny-10k-16v-128px",
    2: "c2-terrain-200k-256v-512px",
    3: "c3-dense-1M-1024v-800px",
    4: "c4-wang-8M-64v-1080p",
    5: "c5-hier-2M-4096v-256px+64v-1024px",
}


def make_scene(cfg: int, n_override: Optional[int] = None, views: Optional[int] = None) -> Scene:
    """BASELINE.json configs[cfg-1].  ``n_override`` / ``views`` shrink a config
    for parity tests (same distributions, fewer draws / fewer cameras)."""
    if cfg == 1:
        fld = gen_config1_field(n_override or 10_000, 0)
        cams = fibonacci_cameras(16, 3.0, 128, 128, 128.0)
        sc = Scene(CONFIG_NAMES[1], fld, cams)
    elif cfg == 2:
        fld = gen_terrain_field(n_override or 200_000, 0, -1.0, 1.0)
        cams = fibonacci_cameras(256, 2.5, 512, 512, 600.0,
                                 math.sin(math.radians(15)), math.sin(math.radians(75)))
        sc = Scene(CONFIG_NAMES[2], fld, cams)
    elif cfg == 3:
        fld = gen_terrain_field(n_override or 1_000_000, 0, -2.0, 2.0)
        cams = fibonacci_cameras(1024, 4.0, 800, 800, 900.0)
        sc = Scene(CONFIG_NAMES[3], fld, cams)
    elif cfg == 4:
        fld = gen_config4_field(n_override or 500_000)
        cams = flyover_cameras(64, 1920, 1080, 1500.0)
        sc = Scene(CONFIG_NAMES[4], fld, cams)
    elif cfg == 5:
        fld = gen_terrain_field(n_override or 2_000_000, 0, -3.0, 3.0)
        cams = fibonacci_cameras(4096, 5.0, 256, 256, 288.0)
        sc = Scene(CONFIG_NAMES[5], fld, cams, fine_width=1024, fine_focal=1152.0, top_k=64)
    else:
        raise ValueError(f"unknown config {cfg}")
    if views is not None:
        sel = np.linspace(0, len(sc.cameras) - 1, views).round().astype(np.int64)
        sc.cameras = np.ascontiguousarray(sc.cameras[sel])
    return sc


def random_scene_small(seed: int, n: int, width: int = 48, height: int = 40, focal: float = 50.0,
                       n_views: int = 3, sh_degree: int = 1, logscale_mu: float = -2.5):
    """Small random scenes for parity edge cases (ragged tiles, several tiles)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    means = rng.uniform(-1.0, 1.0, size=(n, 3))
    scales, q, opac = _activate(rng, n, logscale_mu, 0.5, 0.5, means)
    ncoef = (sh_degree + 1) ** 2
    sh = np.zeros((n, ncoef, 3))
    sh[:, 0, :] = rng.uniform(0.0, 1.0, size=(n, 3))
    if ncoef > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.2, size=(n, ncoef - 1, 3))
    unc = rng.uniform(0.0, 1.0, size=n)
    fld = pack_field(means, scales, q, opac, sh, unc, sh_degree)
    cams = fibonacci_cameras(n_views, 3.0, width, height, focal)
    return fld, cams


# --------------------------------------------------------------------------
# NEXT-1: synthetic diffusion-latent ensembles (VAE
# latents 4 x 64 x 64, M = 5 stochastic passes).  The pretrained prior is not
# available; each candidate view gets a base latent mean, per-sample
# perturbations whose spread varies by view (the "epistemic" signal), and
# per-channel posterior variances.  No method arithmetic here.
# --------------------------------------------------------------------------
def gen_latent_ensembles(n_views: int = 1000, M: int = 5, C: int = 4, H: int = 64, W: int = 64, seed: int = 0):
    """-> (mu, s2) float32 arrays [n_views][M][C][H*W]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    spread = rng.uniform(0.05, 0.5, size=(n_views, 1, 1, 1))
    base = rng.normal(0.0, 1.0, size=(n_views, 1, C, H * W))
    mu = base + spread * rng.normal(0.0, 1.0, size=(n_views, M, C, H * W))
    s2 = np.exp(rng.normal(-2.0, 0.3, size=(n_views, M, C, H * W)))
    return np.ascontiguousarray(mu, dtype=np.float32), np.ascontiguousarray(s2, dtype=np.float32)
