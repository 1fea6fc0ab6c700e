"""Mutation check of the Python oracle modules' pins (the companion of
scripts/oracle_mutants.py, which mutates gsr_oracle.c): for each mutation,
copy the repository's sources to a temporary directory, apply one textual
change to one oracle module there, and run that module's CPU pin suite in
the copy; a mutation must make at least one test fail.

    python scripts/oracle_mutants_py.py

Prints one line per mutation and writes profiles/oracle_mutants_py.json.
Test infrastructure only.
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SKIP = {".git", "gpurun_out", "profiles", "scripts", "__pycache__", ".pytest_cache", "build"}

# (module file, pin suite, name, old text, new text): old occurs exactly once
MUTANTS = [
    ("oracle/w2.py", "tests/test_oracle_w2.py", "W2: no cross term 2 sqrt(s_i s_j)",
     "term += s2[i, c] + s2[j, c] - 2.0 * np.sqrt(s2[i, c] * s2[j, c])", "term += s2[i, c] + s2[j, c]"),
    ("oracle/w2.py", "tests/test_oracle_w2.py", "W2: variances compared as (s2_i - s2_j)^2",
     "term += s2[i, c] + s2[j, c] - 2.0 * np.sqrt(s2[i, c] * s2[j, c])",
     "term += (s2[i, c] - s2[j, c]) ** 2"),
    ("oracle/w2.py", "tests/test_oracle_w2.py", "W2: mean over M^2 ordered pairs",
     "return out / npairs", "return out / (M * M)"),
    ("oracle/sobel.py", "tests/test_oracle_sobel.py", "Sobel: zero instead of replicate padding",
     "rows = np.clip(np.arange(H) + dy, 0, H - 1)", "rows = np.mod(np.arange(H) + dy, H)"),
    ("oracle/sobel.py", "tests/test_oracle_sobel.py", "Sobel: L1 magnitude",
     "return np.sqrt(gx * gx + gy * gy)", "return np.abs(gx) + np.abs(gy)"),
    ("oracle/sobel.py", "tests/test_oracle_sobel.py", "Sobel: y kernel not transposed",
     "gy += SOBEL_X[dx + 1][dy + 1] * v", "gy += SOBEL_X[dy + 1][dx + 1] * v"),
    ("oracle/sobel.py", "tests/test_oracle_sobel.py", "grayscale: sum instead of mean",
     "return (a[..., 0] + a[..., 1] + a[..., 2]) / 3.0", "return a[..., 0] + a[..., 1] + a[..., 2]"),
    ("oracle/optim.py", "tests/test_oracle_optim.py", "Adam: no bias correction of m",
     "mh = m / (1 - beta1 ** t)", "mh = m"),
    ("oracle/optim.py", "tests/test_oracle_optim.py", "Adam: eps inside the sqrt",
     "mh / (np.sqrt(vh) + eps)", "mh / np.sqrt(vh + eps)"),
    ("oracle/optim.py", "tests/test_oracle_optim.py", "L2 loss gradient without the 2",
     "return float((w * d * d).sum() / n), 2.0 * w * d / n", "return float((w * d * d).sum() / n), w * d / n"),
    ("oracle/cache_order.py", "tests/test_oracle_cache_order.py", "cache policy: >= tau",
     "return HOT_BINS if float(u_bar) > tau else BASE_BINS", "return HOT_BINS if float(u_bar) >= tau else BASE_BINS"),
    ("oracle/cache_order.py", "tests/test_oracle_cache_order.py", "cache policy: hot and base swapped",
     "return HOT_BINS if float(u_bar) > tau else BASE_BINS", "return BASE_BINS if float(u_bar) > tau else HOT_BINS"),
    ("oracle/cache_order.py", "tests/test_oracle_cache_order.py", "cached order: descending bin key",
     "out[k] = s + np.lexsort((np.arange(e - s), key))", "out[k] = s + np.lexsort((np.arange(e - s), -key))"),
    ("oracle/cache_order.py", "tests/test_oracle_cache_order.py", "tile visiting order back to front",
     "order = np.lexsort((np.arange(len(centres)), depth))", "order = np.lexsort((np.arange(len(centres)), -depth))"),
    # the backward oracle's float64 forward (pinned against the float32 oracle's image)
    ("oracle/backward.py", "tests/test_oracle_backward.py", "backward forward: j02 sign",
     "j02, j12 = -(fx * tx) / (vz * vz), -(fy * ty) / (vz * vz)", "j02, j12 = (fx * tx) / (vz * vz), -(fy * ty) / (vz * vz)"),
    ("oracle/backward.py", "tests/test_oracle_backward.py", "backward forward: no dilation",
     "a, b, c = Sp[:, 0, 0] + 0.3, Sp[:, 0, 1], Sp[:, 1, 1] + 0.3", "a, b, c = Sp[:, 0, 0], Sp[:, 0, 1], Sp[:, 1, 1]"),
    ("oracle/backward.py", "tests/test_oracle_backward.py", "backward forward: alpha clamp at 1",
     "alpha = torch.clamp(o[g] * torch.exp(power), max=0.99)", "alpha = torch.clamp(o[g] * torch.exp(power), max=1.0)"),
    ("oracle/backward.py", "tests/test_oracle_backward.py", "backward forward: T *= alpha",
     "Tacc = torch.where(mk, Tacc * (1 - alpha), Tacc)", "Tacc = torch.where(mk, Tacc * alpha, Tacc)"),
    ("oracle/backward.py", "tests/test_oracle_backward.py", "backward forward: no colour clamp",
     "rgb = torch.clamp((Y[:, :, None] * P[\"sh\"]).sum(1), min=0.0)", "rgb = (Y[:, :, None] * P[\"sh\"]).sum(1)"),
]


def copy_repo(dst):
    os.makedirs(dst)
    for name in os.listdir(ROOT):
        if name in SKIP:
            continue
        src = os.path.join(ROOT, name)
        if os.path.isdir(src):
            shutil.copytree(src, os.path.join(dst, name), ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        else:
            shutil.copy2(src, os.path.join(dst, name))


def main():
    results = []
    with tempfile.TemporaryDirectory() as td:
        base = os.path.join(td, "base")
        copy_repo(base)
        for mod, suite, name, old, new in MUTANTS:
            src = open(os.path.join(ROOT, mod)).read()
            n = src.count(old)
            if n != 1:
                results.append({"mutation": name, "module": mod, "status": f"SKIPPED (pattern occurs {n}x)"})
                print(results[-1])
                continue
            work = os.path.join(td, "work")
            if os.path.exists(work):
                shutil.rmtree(work)
            shutil.copytree(base, work)
            open(os.path.join(work, mod), "w").write(src.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider", suite],
                               cwd=work, capture_output=True, text=True, timeout=1200)
            failed = [l.split(" ")[1] for l in r.stdout.splitlines() if l.startswith("FAILED")]
            status = "CAUGHT" if r.returncode != 0 else "SURVIVED"
            results.append({"mutation": name, "module": mod, "suite": suite, "status": status,
                            "failing": failed[:5], "n_failing": len(failed)})
            print(f"{status:8s} {name}: {len(failed)} failing" + (f" e.g. {failed[0]}" if failed else ""))
    out = os.path.join(ROOT, "profiles", "oracle_mutants_py.json")
    json.dump(results, open(out, "w"), indent=1)
    print("wrote", out)
    return 0 if all(r["status"] == "CAUGHT" for r in results) else 1


if __name__ == "__main__":
    sys.exit(main())
