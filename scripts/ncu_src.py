"""Per-kernel source-page digest of an ncu report: total warp instructions,
stall samples, and the instruction groups (by execution count) that carry
them.   python scripts/ncu_src.py REPORT KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = None, []
    for r in rows:
        if len(r) > 2 and r[0] == "Address":
            if data:
                break  # first profiled launch only
            hdr = r
            continue
        if hdr and r and r[0].startswith("0x"):
            iS = hdr.index("Warp Stall Sampling (All Samples)")
            iE = hdr.index("Instructions Executed")
            data.append((r[1], int(r[iS] or 0), int(r[iE] or 0)))
    tot = sum(d[2] for d in data)
    tots = sum(d[1] for d in data) or 1
    print(f"{kre}: {tot / 1e6:.1f} M warp-instructions, {tots} stall samples, {len(data)} SASS lines")
    c, s, n = Counter(), Counter(), Counter()
    for src, st, ie in data:
        c[ie] += ie
        s[ie] += st
        n[ie] += 1
    for k in sorted(c, key=lambda k: -c[k])[:top]:
        print(f"  executed {k:10d}x: {n[k]:4d} instrs = {c[k] / 1e6:7.1f} M ({100 * c[k] / tot:4.1f}%), "
              f"stalls {100 * s[k] / tots:4.1f}%")


if __name__ == "__main__":
    main()
