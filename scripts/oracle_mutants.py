"""Mutation check of the oracle pins: compile deliberately wrong copies of
oracle/gsr_oracle.c (one textual mutation each) and run the CPU pin suites
against each; a mutation must make at least one test fail.

    python scripts/oracle_mutants.py [-k PYTEST_EXPR]

Prints one line per mutation (CAUGHT / SURVIVED with the failing tests) and
writes profiles/oracle_mutants.json.  Test infrastructure only.
"""
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "gsr_oracle.c")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_spans.py", "tests/test_oracle_lod.py"]

# (name, old text, new text): each old text must occur exactly once
MUTANTS = [
    ("span margin m = 0", "ORC_SPAN_M = 0.0625f", "ORC_SPAN_M = 0.0f"),
    ("span margin m = 1/4", "ORC_SPAN_M = 0.0625f", "ORC_SPAN_M = 0.25f"),
    ("span ellipse t = 3.33^2", "ORC_SPAN_T = 11.1f", "ORC_SPAN_T = 11.0889f"),
    ("span ellipse t = 3^2", "ORC_SPAN_T = 11.1f", "ORC_SPAN_T = 9.0f"),
    ("span: right extreme at -dys", "float dr = fminf(fmaxf(p->sp_dys, dya), dyb);",
     "float dr = fminf(fmaxf(-p->sp_dys, dya), dyb);"),
    ("span: left extreme at +dys", "float dl = fminf(fmaxf(-p->sp_dys, dya), dyb);",
     "float dl = fminf(fmaxf(p->sp_dys, dya), dyb);"),
    ("span: no band clamp (dr = dys)", "float dr = fminf(fmaxf(p->sp_dys, dya), dyb);", "float dr = p->sp_dys;"),
    ("span: centre line -p dy", "float R = ((p->u + p->sp_p * dr)", "float R = ((p->u - p->sp_p * dr)"),
    ("span: pixel centre not +0.5", "float fpx1 = fminf(floorf(R - 0.5f), (float)(W - 1));",
     "float fpx1 = fminf(floorf(R), (float)(W - 1));"),
    ("SH: direction campos - mu", "float dx = mx - cam->campos[0], dy = my - cam->campos[1], dz = mz - cam->campos[2];",
     "float dx = cam->campos[0] - mx, dy = cam->campos[1] - my, dz = cam->campos[2] - mz;"),
    ("SH: channel-major flat index", "int flat = 3 * k + ch;", "int flat = k + ncoef * ch;"),
    ("SH: no clamp at 0", "rgb[ch] = fmaxf(0.0f, acc);", "rgb[ch] = acc;"),
]


def main():
    src = open(SRC).read()
    kexpr = sys.argv[sys.argv.index("-k") + 1] if "-k" in sys.argv else None
    results = []
    with tempfile.TemporaryDirectory() as td:
        for name, old, new in MUTANTS:
            n = src.count(old)
            if n != 1:
                results.append({"mutation": name, "status": f"SKIPPED (pattern occurs {n}x)"})
                print(results[-1])
                continue
            csrc = os.path.join(td, "m.c")
            lib = os.path.join(td, re.sub(r"\W+", "_", name) + ".so")
            open(csrc, "w").write(src.replace(old, new))
            subprocess.check_call(["gcc", *CFLAGS, "-o", lib, csrc, "-lm", "-lpthread"])
            env = dict(os.environ, GSR_ORACLE_LIB=lib)
            cmd = [sys.executable, "-m", "pytest", "-q", "-x" if False else "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                   *TESTS] + (["-k", kexpr] if kexpr else [])
            r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True)
            failed = sorted(set(re.findall(r"FAILED (\S+)", r.stdout)))
            status = "CAUGHT" if r.returncode != 0 else "SURVIVED"
            results.append({"mutation": name, "status": status, "failed": failed})
            print(f"{status:8s} {name}: {len(failed)} failing" + (f" e.g. {failed[0]}" if failed else ""), flush=True)
    out = os.path.join(ROOT, "profiles", "oracle_mutants.json")
    json.dump(results, open(out, "w"), indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
