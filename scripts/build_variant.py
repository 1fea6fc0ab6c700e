"""Build an A/B variant of libgsr with extra -D flags (GSR_LIB selects it):

    python scripts/build_variant.py libgsr_k3ls0.so -DK3_LS=0
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_15355_b200 import build as B  # noqa: E402

out = os.path.join(B.HERE, sys.argv[1])
cmd = [B.NVCC, *B.NVCC_FLAGS, *sys.argv[2:], "-shared", "-o", out, *B.sources(),
       "-Xlinker", "--version-script=" + os.path.join(B.CSRC, "exports.map")]
subprocess.check_call(cmd)
print(out)
