"""Small hand-built inputs for the pins (no method arithmetic here)."""
import numpy as np

import synth


def axis_camera(width, height, focal, cx=None, cy=None, znear=0.2):
    """Camera at the origin looking down +z (R = I, t = 0), OpenCV axes."""
    cam = np.zeros((), dtype=synth.CAM_DTYPE)
    cam["R"] = np.eye(3, dtype=np.float32).reshape(-1)
    cam["t"] = 0.0
    cam["campos"] = 0.0
    cam["fx"] = focal
    cam["fy"] = focal
    cam["cx"] = width / 2.0 if cx is None else cx
    cam["cy"] = height / 2.0 if cy is None else cy
    cam["limx"] = np.float32(1.3 * (width / 2.0) / focal)
    cam["limy"] = np.float32(1.3 * (height / 2.0) / focal)
    cam["znear"] = znear
    cam["width"] = width
    cam["height"] = height
    return cam


def field_from(means, scales, quats, opac, rgb, unc, sh_degree=0, sh_rest=None):
    means = np.atleast_2d(np.asarray(means, dtype=np.float64))
    n = len(means)
    ncoef = (sh_degree + 1) ** 2
    sh = np.zeros((n, ncoef, 3))
    sh[:, 0, :] = np.asarray(rgb, dtype=np.float64).reshape(n, 3)
    if sh_rest is not None:
        sh[:, 1:, :] = sh_rest
    return synth.pack_field(means, np.asarray(scales, np.float64).reshape(n, 3),
                            np.asarray(quats, np.float64).reshape(n, 4),
                            np.asarray(opac, np.float64).reshape(n),
                            sh, np.asarray(unc, np.float64).reshape(n), sh_degree)


def random_unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)
