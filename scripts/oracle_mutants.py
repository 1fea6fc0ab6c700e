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

# (name, old text, new text[, "all"]): the old text must occur exactly once,
# or, tagged "all", every occurrence is replaced (the same rule in two loops)
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
    # exp_spec (O5 note)
    ("exp: no ln2_lo correction", "r = fmaf(kf, -ln2_lo, r);", "(void)ln2_lo;"),
    ("exp: 2^k off by one", "float scale = u2f((uint32_t)(k + 127) << 23);",
     "float scale = u2f((uint32_t)(k + 128) << 23);"),
    ("exp: 1/6! term dropped", "p = fmaf(p, r, u2f(0x3ab60b61u));", "p = fmaf(p, r, 0.0f);"),
    # projection (O1)
    ("EWA: no 0.3 px^2 dilation", "static const float ORC_DILATION = 0.3f;", "static const float ORC_DILATION = 0.0f;"),
    ("EWA: no FOV clamp in x", "float tx = fminf(cam->limx, fmaxf(-cam->limx, xn)) * vz;", "float tx = xn * vz;"),
    ("Jacobian: j02 sign", "float j02 = -(cam->fx * tx) / z2;", "float j02 = (cam->fx * tx) / z2;"),
    ("quaternion: R01 sign", "rm[0][1] = 2.0f * (x * y - w * z);", "rm[0][1] = 2.0f * (x * y + w * z);"),
    ("Sigma = M^T M", "S[i][j] = (M[i][0] * M[j][0] + M[i][1] * M[j][1]) + M[i][2] * M[j][2];",
     "S[i][j] = (M[0][i] * M[0][j] + M[1][i] * M[1][j]) + M[2][i] * M[2][j];"),
    ("near cull at 0 instead of znear", "if (!(vz > cam->znear)) return;", "if (!(vz > 0.0f)) return;"),
    # compositing (O5) and score (O6)
    ("alpha clamp 1.0", "static const float ORC_ALPHA_MAX = 0.99f;", "static const float ORC_ALPHA_MAX = 1.0f;"),
    ("T stop 1e-3", "static const float ORC_T_STOP = 1e-4f;", "static const float ORC_T_STOP = 1e-3f;"),
    ("no alpha < 1/255 skip", "static const float ORC_ALPHA_MIN = 1.0f / 255.0f;",
     "static const float ORC_ALPHA_MIN = 0.0f;"),
    ("power: + B dx dy", "float power = fmaf(-0.5f, qf, -((q->B * dx) * dy));",
     "float power = fmaf(-0.5f, qf, ((q->B * dx) * dy));", "all"),
    ("no early stop", "if (tT < ORC_T_STOP) { *n_eval = (uint64_t)(i + 1); break; }",
     "if (tT < 0.0f) { *n_eval = (uint64_t)(i + 1); break; }"),
    ("score from red instead of U", "sum += (double)o4[3];", "sum += (double)o4[0];", "all"),
    ("score over W*H-1 pixels", "return sum / ((double)W * (double)H);", "return sum / ((double)W * (double)H - 1.0);",
     "all"),
]


def main():
    src = open(SRC).read()
    kexpr = sys.argv[sys.argv.index("-k") + 1] if "-k" in sys.argv else None
    results = []
    with tempfile.TemporaryDirectory() as td:
        for name, old, new, *mode in MUTANTS:
            n = src.count(old)
            if n != 1 and not (mode and mode[0] == "all" and n > 1):
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
