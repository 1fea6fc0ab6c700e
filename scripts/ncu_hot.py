"""Summarise an ncu source page CSV: hottest SASS lines by stall samples."""
import csv
import sys

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
which = sys.argv[3] if len(sys.argv) > 3 else None  # substring of the kernel name
rows = list(csv.reader(open(path)))
# the file may hold several kernels: split at "Kernel Name" rows
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sel = [b for b in blocks if which is None or which in b["name"]][:1]
for b in sel:
    hdr, data = b["rows"][0], b["rows"][1:]
    i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    i_e, i_t = hdr.index("Instructions Executed"), hdr.index("Avg. Threads Executed")
    tot = sum(int(r[i_s]) for r in data) or 1
    tote = sum(int(r[i_e]) for r in data) or 1
    print(b["name"][:120])
    print("samples", tot, "warp-inst", tote, "sass lines", len(data))
    hot = sorted(range(len(data)), key=lambda k: -int(data[k][i_s]))[:top]
    for k in sorted(hot):
        r = data[k]
        print(f"{k:4d} {int(r[i_s]) / tot * 100:5.1f}% inst={int(r[i_e]) / tote * 100:5.1f}% thr={r[i_t]:>5} {r[i_src][:80]}")
