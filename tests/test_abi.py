"""CPU-side checks of the C ABI: the library loads and exports every symbol
include/gsr.h declares; host-only logic (the camera builder) matches the
input generator; struct layouts match the header.  No GPU compute here."""
import ctypes
import math
import os
import re

import numpy as np

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gsr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2602_15355_b200 import gsr
    names = declared_symbols()
    assert len(names) >= 12
    lib = ctypes.CDLL(gsr.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(gsr.EXPORTED)
    assert gsr.version().startswith("gsr ")


def test_camera_layout_matches_header_and_generator():
    from paper_2602_15355_b200 import gsr
    assert gsr.CAM_DTYPE.itemsize == 96 == synth.CAM_DTYPE.itemsize
    assert gsr.CAM_DTYPE.names == synth.CAM_DTYPE.names
    assert ctypes.sizeof(gsr._Gaussians) == 48


def test_camera_look_at_host_builder_matches_generator():
    """gsr_camera_look_at (C, double) == synth.camera_from_theta (numpy, double),
    both rounded once to float32: equal within 1 ulp."""
    from paper_2602_15355_b200 import gsr
    rng = np.random.default_rng(0)
    for _ in range(50):
        e, a, r = rng.uniform(0.05, 1.5), rng.uniform(0, 2 * math.pi), rng.uniform(1, 6)
        tgt = rng.uniform(-1, 1, 3)
        c = gsr.gsr_camera_look_at(e, a, r, tgt, 640, 480, 500.0, 0.2)
        s = synth.camera_from_theta(e, a, r, 640, 480, 500.0, target=tgt)
        for f in ("R", "t", "campos"):
            x, y = np.asarray(c[f], np.float32), np.asarray(s[f], np.float32)
            assert np.all(np.abs(x - y) <= 2 * np.spacing(np.maximum(np.abs(x), np.abs(y)))), f
        for f in ("fx", "fy", "cx", "cy", "limx", "limy", "znear", "width", "height"):
            assert c[f] == s[f], f


def test_camera_look_at_rejects_bad_arguments():
    import pytest
    from paper_2602_15355_b200 import gsr
    with pytest.raises(gsr.GsrError) as ei:
        gsr.gsr_camera_look_at(0.3, 0.1, 2.0, [0, 0, 0], 0, 10, 100.0)
    assert ei.value.status == gsr.GSR_EINVAL
    with pytest.raises(gsr.GsrError):
        gsr.gsr_camera_look_at(0.3, 0.1, -2.0, [0, 0, 0], 10, 10, 100.0)
