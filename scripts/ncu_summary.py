"""Summarise ncu outputs into profiles/ (tracked):

    python scripts/ncu_summary.py TAG gpurun_out/launches_TAG.csv gpurun_out/prof_TAG.ncu-rep

writes profiles/TAG_launches.csv (kernel, launches, total/avg device time,
share of the step) and profiles/TAG_ncu.json / .md (per profiled kernel: time,
DRAM bytes read+write, achieved DRAM GB/s, issue/warp utilisation, registers,
occupancy limiters).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    n = name.replace("CUtensorMap_st, ", "").replace("void ", "").replace("gsr::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    n = n.replace("unnamed>::", "")
    for sep in ("(const", "(float", "(unsigned", "(long", "(int"):
        if sep in n:
            n = n[: n.index(sep)]
    return n.strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "nsecond"
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values()) or 1.0
    out = [(k, a[0], a[1] / 1e3, a[1] / a[0] / 1e3, a[1] / tot) for k, a in agg.items()]
    return sorted(out, key=lambda x: -x[2])


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = {
        "time_ms": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum", "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "regs": "launch__registers_per_thread", "grid": "launch__grid_size", "block": "launch__block_size",
        "occ_limit_regs": "launch__occupancy_limit_registers", "occ_limit_smem": "launch__occupancy_limit_shared_mem",
        "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l2_bytes": "lts__t_bytes.sum", "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "warp_inst": "smsp__inst_executed.sum",
    }
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
             "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    res = []
    for r in data:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, m in want.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if k.startswith("dram_r") or k.startswith("dram_w") or k == "l2_bytes":
                v *= scale.get(u, 1)
            if k == "time_ms":
                v *= scale.get(u, 1)
            d[k] = v
        if "dram_read" in d and "time_ms" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
            d["dram_GBps"] = d["dram_bytes"] / (d["time_ms"] * 1e-3) / 1e9
        res.append(d)
    return res


def main():
    tag, lpath, rep = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None
    os.makedirs(PROF, exist_ok=True)
    L = launches(lpath)
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_us", "avg_us", "share_of_listed_time"])
        for k, n, t, a, s in L:
            w.writerow([k, n, f"{t:.1f}", f"{a:.2f}", f"{s:.4f}"])
    md = [f"# ncu summary {tag}", "", "## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache,"
          " serialised: compare shares)", "", "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    md += [f"| {k} | {n} | {t:.1f} | {a:.2f} | {s:.1%} |" for k, n, t, a, s in L]
    if rep and os.path.exists(rep):
        R = ncu_raw(rep)
        json.dump(R, open(os.path.join(PROF, f"{tag}_ncu.json"), "w"), indent=1)
        md += ["", "## ncu --set full (per profiled launch)", "",
               "| kernel | ms | DRAM MB (r+w) | DRAM GB/s | issue % | warps % | FMA pipe % | regs |",
               "|---|---|---|---|---|---|---|---|"]
        for d in R:
            md.append(f"| {d['kernel']} | {d.get('time_ms', 0):.3f} | {d.get('dram_bytes', 0) / 1e6:.1f} | "
                      f"{d.get('dram_GBps', 0):.0f} | {d.get('issue_active_pct', 0):.1f} | "
                      f"{d.get('warps_active_pct', 0):.1f} | {d.get('fma_pipe_pct', 0):.1f} | {d.get('regs', 0):.0f} |")
    open(os.path.join(PROF, f"{tag}_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
