"""Mutation check of the GPU parity tests: build libgsr.so copies with one
deliberate textual change each in the CUDA sources (the kind of slip a kernel
edit can make), then run the parity suites against each copy on the GPU;
every mutation must make a test fail.

    python scripts/kernel_mutants.py build    # here: scripts/scratch/mut_*.so + manifest
    python scripts/kernel_mutants.py run      # on the GPU box: writes gpurun_out/kernel_mutants.json

Test infrastructure only (the product library is never modified).
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "scripts", "scratch")
SUITES = ["tests/test_gpu_parity.py", "tests/test_gpu_adversarial.py"]

# (name, file under csrc/, old text, new text): old occurs exactly once
MUTANTS = [
    ("K1: no SH colour clamp", "project.cu", "rgb[ch] = fmaxf(0.0f, acc);", "rgb[ch] = acc;"),
    ("K1: tau not stored (record word 7 = o)", "project.cu", "rr[1] = make_float4(C, o, Sd.w, tau);",
     "rr[1] = make_float4(C, o, Sd.w, -1.0e30f);"),
    ("spans: tile range end not +1", "gsr_internal.cuh", "x1 = ((uint32_t)fx1 >> 4) + 1u;",
     "x1 = ((uint32_t)fx1 >> 4);"),
    ("K4c: ranks counted from the top", "binsort.cu", "rk[k] = pre + __popc(peers & lt);",
     "rk[k] = pre + __popc(peers & ~lt & ~(1u << lane));"),
    ("K6: alpha clamp at 1 for the first hit of a pair", "composite.cu",
     "const float alpha_a = fminf(kAlphaMax, lo2(al)), alpha_b = fminf(kAlphaMax, hi2(al));",
     "const float alpha_a = fminf(1.0f, lo2(al)), alpha_b = fminf(kAlphaMax, hi2(al));"),
    ("K6: odd hit count not padded", "composite.cu",
     "reinterpret_cast<float*>(&s_pr[warp][nh >> 1][2])[3] = __int_as_float(0x7f800000);",
     "(void)0;"),
    ("K6: box cull without slack", "composite.cu", "hit = qmin <= (-2.0f * r1.w) * 1.001f + 1e-3f;",
     "hit = qmin <= (-2.0f * r1.w) * 0.999f - 1e-3f;"),
    ("exp: 1/6! coefficient (packed path)", "composite.cu",
     "f32x2 p = ffma2(bc2(c7), r, bc2(__int_as_float(0x3ab60b61)));",
     "f32x2 p = ffma2(bc2(c7), r, bc2(__int_as_float(0x3ab60b62)));"),
    ("K7: score not divided by the pixel count", "composite.cu", "scores[v] = (float)(t * inv_area);",
     "scores[v] = (float)t;"),
]


def build():
    sys.path.insert(0, os.path.join(ROOT, "paper_2602_15355_b200"))
    import build as B
    os.makedirs(OUT, exist_ok=True)
    manifest = []
    procs = []
    for i, (name, fn, old, new) in enumerate(MUTANTS):
        td = tempfile.mkdtemp(prefix="mut")
        srcs = []
        for s in B.sources() + [os.path.join(B.CSRC, "gsr_internal.cuh")]:
            dst = os.path.join(td, os.path.basename(s))
            txt = open(s).read()
            if os.path.basename(s) == fn:
                assert txt.count(old) == 1, (name, txt.count(old))
                txt = txt.replace(old, new)
            txt = txt.replace('"../../include/gsr.h"', '"' + os.path.join(ROOT, "include", "gsr.h") + '"')
            open(dst, "w").write(txt)
            if dst.endswith(".cu"):
                srcs.append(dst)
        lib = os.path.join(OUT, f"mut_{i}.so")
        cmd = [B.NVCC, *B.NVCC_FLAGS, "-shared", "-o", lib, *srcs,
               "-Xlinker", "--version-script=" + os.path.join(B.CSRC, "exports.map")]
        procs.append(subprocess.Popen(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.PIPE))
        manifest.append({"mutation": name, "file": fn, "lib": os.path.relpath(lib, ROOT)})
    for p, m in zip(procs, manifest):
        _, err = p.communicate()
        assert p.returncode == 0, (m, err.decode()[-2000:])
    json.dump(manifest, open(os.path.join(OUT, "mut_manifest.json"), "w"), indent=1)
    print("built", len(manifest))


def run():
    manifest = json.load(open(os.path.join(OUT, "mut_manifest.json")))
    res = []
    for m in manifest:
        env = dict(os.environ, GSR_LIB=os.path.join(ROOT, m["lib"]))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", *SUITES],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
        failed = [l.split(" ")[1] for l in r.stdout.splitlines() if l.startswith("FAILED")]
        status = "CAUGHT" if r.returncode != 0 else "SURVIVED"
        res.append({"mutation": m["mutation"], "file": m["file"], "status": status, "n_failing": len(failed),
                    "failing": failed[:5]})
        print(f"{status:8s} {m['mutation']}: {len(failed)} failing" + (f" e.g. {failed[0]}" if failed else ""),
              flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "kernel_mutants.json"), "w"), indent=1)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
