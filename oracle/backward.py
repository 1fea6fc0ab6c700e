"""NEXT-3 oracle: gradients of the rendered view w.r.t. the Gaussian
parameters -- the backward rasterizer that UPDATE_GS needs (Alg. 1
L158 "incremental Gaussian-splat updates", §4.1 L302 refinement) -- TEST
INFRASTRUCTURE ONLY (same rules as the package docstring of oracle/).

Plain PyTorch CPU float64 autograd of the O1 / O4 / O5 forward written with
torch ops in the order of SURVEY §8(c), with the forward's discrete structure
frozen: which (pixel, Gaussian) pairs are blended, and in which order, comes
from the float32 oracle (``composite_trace``) -- the same decisions the CUDA
forward makes bit for bit.  Between those decisions the image is a smooth
function of the parameters, and this module differentiates it exactly (up to
float64 rounding).  The loss is the linear functional L = sum_p <G_p, C_p>
of the composited (r, g, b, U) image C with an upstream gradient G, so the
result is the vector-Jacobian product a training step needs for any loss.

Parameters follow the field's plane layout (synth.pack_field): means,
activated scales, raw quaternion (normalised inside, as K1 does), activated
opacity (times the LOD weight when blending is on: a constant per view),
uncertainty, SH coefficients (DC = colour).  Output: float64 [P][n][4] in
the same layout.  Pins: tests/test_oracle_backward.py (central finite
differences of this forward, closed forms for one Gaussian).
"""
from __future__ import annotations

import numpy as np
import torch

from . import bin_sort_batch, composite_trace, lod_weight, project

SH_C = dict(C1=0.4886025119, C2a=1.0925484306, C2b=0.3153915653, C2c=0.5462742153, C3a=0.5900435899,
            C3b=2.8906114426, C3c=0.4570457995, C3d=0.3731763326, C3e=1.4453057213)


def sh_basis_t(d, deg):
    """O4 real SH basis (Y0 = 1) of unit directions d [n][3] (torch)."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    Y = [torch.ones_like(x)]
    if deg >= 1:
        Y += [-SH_C["C1"] * y, SH_C["C1"] * z, -SH_C["C1"] * x]
    if deg >= 2:
        xx, yy, zz = x * x, y * y, z * z
        Y += [SH_C["C2a"] * x * y, -SH_C["C2a"] * y * z, SH_C["C2b"] * (2 * zz - xx - yy), -SH_C["C2a"] * x * z,
              SH_C["C2c"] * (xx - yy)]
    if deg >= 3:
        Y += [-SH_C["C3a"] * y * (3 * xx - yy), SH_C["C3b"] * x * y * z, -SH_C["C3c"] * y * (4 * zz - xx - yy),
              SH_C["C3d"] * z * (2 * zz - 3 * xx - 3 * yy), -SH_C["C3c"] * x * (4 * zz - xx - yy),
              SH_C["C3e"] * z * (xx - yy), -SH_C["C3a"] * x * (xx - 3 * yy)]
    return torch.stack(Y, 1)


def params_from_field(field):
    """float64 leaf tensors (requires_grad) from the float32 planes."""
    pl = torch.from_numpy(np.asarray(field.planes, dtype=np.float64))
    n, deg = field.n, field.sh_degree
    K = (deg + 1) ** 2
    flat = pl[3:].permute(1, 0, 2).reshape(n, -1)[:, :3 * K]
    P = dict(means=pl[0, :, :3], opac=pl[0, :, 3], scales=pl[1, :, :3], unc=pl[1, :, 3], quats=pl[2],
             sh=flat.reshape(n, K, 3))
    return {k: v.clone().requires_grad_(True) for k, v in P.items()}


def project_t(P, cam, deg, opac_scale=None):
    """O1 + O4 in float64 torch for all Gaussians: u, v, conic A, B, C,
    opacity, colour (r, g, b, U)."""
    f = lambda k: torch.tensor(np.float64(np.float32(cam[k])))  # noqa: E731
    R = torch.from_numpy(np.asarray(cam["R"], dtype=np.float64).reshape(3, 3))
    t = torch.from_numpy(np.asarray(cam["t"], dtype=np.float64))
    campos = torch.from_numpy(np.asarray(cam["campos"], dtype=np.float64))
    fx, fy, cx, cy, limx, limy = f("fx"), f("fy"), f("cx"), f("cy"), f("limx"), f("limy")
    m = P["means"]
    vc = m @ R.T + t
    vx, vy, vz = vc[:, 0], vc[:, 1], vc[:, 2]
    xn, yn = vx / vz, vy / vz
    u, v = fx * xn + cx, fy * yn + cy
    q = P["quats"] / torch.linalg.norm(P["quats"], dim=1, keepdim=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    Rq = torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1),
        torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1),
        torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)], 1)
    M = Rq * P["scales"][:, None, :]
    Sig = M @ M.transpose(1, 2)
    tx = torch.clamp(xn, -limx, limx) * vz
    ty = torch.clamp(yn, -limy, limy) * vz
    j00, j11 = fx / vz, fy / vz
    j02, j12 = -(fx * tx) / (vz * vz), -(fy * ty) / (vz * vz)
    T0 = j00[:, None] * R[0][None, :] + j02[:, None] * R[2][None, :]
    T1 = j11[:, None] * R[1][None, :] + j12[:, None] * R[2][None, :]
    T = torch.stack([T0, T1], 1)
    Sp = T @ Sig @ T.transpose(1, 2)
    a, b, c = Sp[:, 0, 0] + 0.3, Sp[:, 0, 1], Sp[:, 1, 1] + 0.3
    det = a * c - b * b
    A, B, C = c / det, -b / det, a / det
    d = m - campos
    d = d / torch.linalg.norm(d, dim=1, keepdim=True)
    Y = sh_basis_t(d, deg)
    rgb = torch.clamp((Y[:, :, None] * P["sh"]).sum(1), min=0.0)
    o = P["opac"] if opac_scale is None else P["opac"] * opac_scale
    col = torch.cat([rgb, P["unc"][:, None]], 1)
    return u, v, A, B, C, o, col


def render_t(P, cam, deg, off, idx, opac_scale=None):
    """O5 over the frozen blend lists (off, idx) -> C [H][W][4] (float64 torch)."""
    u, v, A, B, C, o, col = project_t(P, cam, deg, opac_scale)
    W, H = int(cam["width"]), int(cam["height"])
    cnt = np.diff(off)
    mx = int(cnt.max()) if len(cnt) else 0
    npx = W * H
    Cimg = torch.zeros(npx, 4, dtype=torch.float64)
    if mx == 0:
        return Cimg.reshape(H, W, 4)
    gi = np.zeros((npx, mx), dtype=np.int64)
    mask = np.zeros((npx, mx), dtype=bool)
    for k in range(mx):
        has = cnt > k
        gi[has, k] = idx[off[:-1][has] + k]
        mask[:, k] = has
    pix = np.arange(npx)
    pcx = torch.from_numpy((pix % W).astype(np.float64) + 0.5)
    pcy = torch.from_numpy((pix // W).astype(np.float64) + 0.5)
    Tacc = torch.ones(npx, dtype=torch.float64)
    for k in range(mx):
        g = torch.from_numpy(gi[:, k])
        mk = torch.from_numpy(mask[:, k])
        dx, dy = u[g] - pcx, v[g] - pcy
        power = -0.5 * (A[g] * dx * dx + C[g] * dy * dy) - B[g] * dx * dy
        alpha = torch.clamp(o[g] * torch.exp(power), max=0.99)
        wgt = torch.where(mk, alpha * Tacc, torch.zeros_like(Tacc))
        Cimg = Cimg + wgt[:, None] * col[g]
        Tacc = torch.where(mk, Tacc * (1 - alpha), Tacc)
    return Cimg.reshape(H, W, 4)


def lod_scale(field_n, cam, lod):
    """Per-Gaussian LOD weights at this camera (constants of the backward),
    computed by the float32 oracle's own O1 LOD rule."""
    if lod is None:
        return None
    campos = np.asarray(cam["campos"], dtype=np.float32)
    tl = lod.tile_level
    d = np.sqrt(((campos[0] - tl[:, 0]) * (campos[0] - tl[:, 0]) + (campos[1] - tl[:, 1]) * (campos[1] - tl[:, 1]))
                + (campos[2] - tl[:, 2]) * (campos[2] - tl[:, 2])).astype(np.float32)
    return torch.tensor([lod_weight(d[i], int(tl[i, 3]), lod) for i in range(field_n)], dtype=torch.float64)


def frozen_lists(field, cam, lod=None):
    """The float32 forward's blend lists of one view (composite_trace)."""
    p = project(field, cam, lod)
    bs = bin_sort_batch([p], np.asarray([cam]))
    return composite_trace(p, bs["vals"], bs["ranges"], cam)


def pack_grads(P, n, deg):
    """Gradients in the plane layout [3 + ceil(3 (deg+1)^2 / 4)][n][4]."""
    K = (deg + 1) ** 2
    nsh = (3 * K + 3) // 4
    out = np.zeros((3 + nsh, n, 4), dtype=np.float64)
    g = {k: (v.grad.numpy() if v.grad is not None else np.zeros(v.shape)) for k, v in P.items()}
    out[0, :, :3], out[0, :, 3] = g["means"], g["opac"]
    out[1, :, :3], out[1, :, 3] = g["scales"], g["unc"]
    out[2] = g["quats"]
    flat = np.zeros((n, 4 * nsh))
    flat[:, :3 * K] = g["sh"].reshape(n, 3 * K)
    out[3:] = flat.reshape(n, nsh, 4).transpose(1, 0, 2)
    return out


def backward_views(field, cams, G, lod=None):
    """Sum over the views of dL/dparams with L = sum_v sum_p <G[v, p], C_v(p)>;
    G: [V][H][W][4].  Returns float64 [P][n][4]."""
    P = params_from_field(field)
    total = None
    for vi, cam in enumerate(cams):
        off, idx = frozen_lists(field, cam, lod)
        img = render_t(P, cam, field.sh_degree, off, idx, lod_scale(field.n, cam, lod))
        L = (img * torch.from_numpy(np.asarray(G[vi], dtype=np.float64))).sum()
        total = L if total is None else total + L
    total.backward()
    return pack_grads(P, field.n, field.sh_degree)
