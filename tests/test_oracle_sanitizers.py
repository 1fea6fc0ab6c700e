"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY.md
§4.2 level 4, §5): gsr_oracle.c is rebuilt with
-fsanitize=address,undefined (UB fatal) and the oracle's pin suites run
against that build in a subprocess (libasan / libubsan preloaded into the
Python interpreter, which loads the oracle through ctypes).  Any
out-of-bounds access, use-after-free, overflow or invalid shift fails it.
The GPU side has no sanitizer on this pool (compute-sanitizer is closed
there); its counterpart is the GSR_DEBUG build's device bounds checks
(tests/test_gpu_debug_build.py)."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_oracle_pins.py", "tests/test_oracle_spans.py", "tests/test_oracle_lod.py",
          "tests/test_oracle_cache_order.py"]


def _runtime(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


@pytest.mark.skipif(shutil.which("gcc") is None or _runtime("libasan.so") is None, reason="no gcc / libasan")
def test_oracle_pins_under_asan_ubsan(tmp_path):
    lib = tmp_path / "liboracle_asan.so"
    subprocess.check_call(["gcc", "-O1", "-g", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                           "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
                           "-fno-omit-frame-pointer", "-o", str(lib), os.path.join(ROOT, "oracle", "gsr_oracle.c"),
                           "-lm", "-lpthread"])
    env = dict(os.environ, GSR_ORACLE_LIB=str(lib), ASAN_OPTIONS="detect_leaks=0:abort_on_error=0",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1",
               LD_PRELOAD=":".join(p for p in (_runtime("libasan.so"), _runtime("libubsan.so")) if p))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider", *SUITES],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "AddressSanitizer" not in out and "runtime error" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert " passed" in r.stdout
