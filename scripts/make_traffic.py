"""profiles/traffic.json from a committed ncu summary (scripts/ncu_summary.py
output): DRAM read+write bytes per launch of K6 and of the K4c tile sort
(cs_hist + cs_scan + cs_scatter of one batch), and K6's pipe fractions, which
bench.py reports as roofline.traffic / roofline.ncu when the batch size
matches.   python scripts/make_traffic.py TAG [VIEWS_PER_LAUNCH]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    tag = sys.argv[1]
    views = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    R = json.load(open(os.path.join(ROOT, "profiles", f"{tag}_ncu.json")))
    first = {}
    for d in R:  # the first profiled launch of each kernel
        first.setdefault(d["kernel"], d)
    k6 = next(v for k, v in first.items() if k.startswith("k6_composite"))
    ts = sum(v["dram_bytes"] for k, v in first.items() if k in ("cs_hist", "cs_scan") or k.startswith("cs_scatter"))
    out = {"k6_composite": k6["dram_bytes"], "tile_sort": ts, "views_per_launch": views,
           "k6_ncu": {"issue_active_pct": round(k6.get("issue_active_pct", 0), 1),
                      "fma_pipe_pct": round(k6.get("fma_pipe_pct", 0), 1),
                      "alu_pipe_pct": round(k6.get("alu_pipe_pct", 0), 1),
                      "warps_active_pct": round(k6.get("warps_active_pct", 0), 1),
                      "warp_inst": k6.get("warp_inst"),
                      "_metrics": f"smsp__issue_active, sm__pipe_fma_cycles_active, sm__inst_executed_pipe_alu, "
                                  f"sm__warps_active (pct_of_peak_sustained_active), smsp__inst_executed.sum; "
                                  f"profiles/{tag} ncu --set full"},
           "_source": f"profiles/{tag}_ncu.json (ncu --set full, --clock-control none, bench.py --slots 1, "
                      f"{views}-view batches): DRAM read+write bytes per K6 launch and per K4c tile sort "
                      f"(cs_hist + cs_scan + cs_scatter)"}
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
