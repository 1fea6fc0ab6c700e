"""The GPU path under its debug build (libgsr_debug.so: -DGSR_DEBUG, device
bounds checks GSR_DCHECK on every computed global index of K2, K3, the
onesweep passes, K4c, K6 and K6b; a violation traps).  compute-sanitizer is
closed on this pool, so this is the memory-safety evidence for the kernels:
the parity suites and the sanitize_run driver (every default kernel plus
the 64-bit depth-key and radix tile-sort fallbacks) run in a subprocess
against the debug library and must pass with no trap."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _debug_lib():
    sys.path.insert(0, os.path.join(ROOT, "paper_2602_15355_b200"))
    import importlib.util
    spec = importlib.util.spec_from_file_location("_gsr_build", os.path.join(ROOT, "paper_2602_15355_b200", "build.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    return B.build(debug=True)


def test_parity_and_all_kernels_under_device_bounds_checks():
    lib = _debug_lib()
    assert lib.endswith("libgsr_debug.so") and os.path.exists(lib)
    env = dict(os.environ, GSR_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py"), "--variants"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.count("sanitize_run ok") == 2, (r.stdout + r.stderr)[-3000:]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_adversarial.py", "tests/test_gpu_backward.py",
                        "tests/test_gpu_lod.py", "tests/test_gpu_cache_order.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert "GSR_DCHECK failed" not in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]


_TRAP_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import synth
from paper_2602_15355_b200 import Context, gsr
from tests.gpu_utils import gpu_batch, to_dev
from tests.helpers import axis_camera
sc = synth.make_scene(1, n_override=500, views=2)
cams = np.stack([axis_camera(32, 32, 32.0)] * 2)
ctx = Context(0)
g = gpu_batch(ctx, sc.field, cams, images=False, want_unsorted=False, want_keys=False)
rec = torch.zeros((2, 500, 12), device="cuda")
vals = torch.from_numpy(g["vals"].astype(np.int32)).cuda()
vals[:] = 500  # every list entry names a Gaussian past the end of the records
ranges = torch.from_numpy(g["ranges"].astype(np.int32).reshape(-1, 2)).cuda()
part = torch.zeros(ranges.shape[0], device="cuda")
try:
    gsr.gsr_composite(ctx, rec, 500, vals, ranges, cams, part)
    torch.cuda.synchronize()
except Exception as e:
    print("trapped:", type(e).__name__, e)
    sys.exit(3)
print("no trap")
"""


def test_debug_checks_trap_on_a_bad_index(tmp_path):
    """The checks are live: composite lists naming Gaussians past the end of
    the render records trap (GSR_DCHECK(g < n) in K6) instead of reading
    out of bounds."""
    lib = _debug_lib()
    f = tmp_path / "trap_child.py"
    f.write_text(_TRAP_CHILD)
    r = subprocess.run([sys.executable, str(f), ROOT], cwd=ROOT, env=dict(os.environ, GSR_LIB=lib),
                       capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert r.returncode == 3 and "trapped:" in out, out[-2000:]
