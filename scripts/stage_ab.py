"""Single-stream per-stage device times of the c3 scoring pass, A/B over
environment settings (each setting in its own process: libgsr reads its
GSR_* switches at context creation).

    python scripts/stage_ab.py [--views 256] "" "GSR_TSORT=cs" ...

Prints one JSON line per setting: ms per 32-view batch for every stage (CUDA
events on the launching stream, one slot, after a warm-up pass) and the
stage's algorithmic GB/s.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(views: int, slots: int):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    import synth
    from paper_2602_15355_b200 import Gaussians
    from paper_2602_15355_b200.pipeline import ViewScorer

    sc = synth.make_scene(3)
    G = Gaussians(torch.from_numpy(sc.field.planes).cuda(), sc.field.sh_degree)
    cams = sc.cameras[:: max(1, len(sc.cameras) // views)][:views]
    s = ViewScorer(G, batch_views=32, n_slots=slots)
    s.count_fragments = False  # as bench.py times it
    s.score_views(cams)
    torch.cuda.synchronize()
    s.timing(True)
    s.timing_read()
    s.reset_counters()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    scores = s.score_views(cams)
    ev1.record()
    torch.cuda.synchronize()
    st = s.timing_read()
    nb = views / 32
    out = {"env": os.environ.get("AB_TAG", ""), "views": views, "slots": slots,
           "pass_ms_per_batch": round(ev0.elapsed_time(ev1) / nb, 4),
           "score_sum": float(scores.double().sum().item())}
    for k, v in st.items():
        if v["launches"]:
            out[k] = {"ms": round(v["ms"] / nb, 4),
                      "GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else None}
    out["sum_ms"] = round(sum(v["ms"] for v in st.values()) / nb, 4)
    print(json.dumps(out), flush=True)


def main():
    args = sys.argv[1:]
    views, slots = 256, 1
    if args[:1] == ["--views"]:
        views, args = int(args[1]), args[2:]
    if args[:1] == ["--slots"]:
        slots, args = int(args[1]), args[2:]
    if args and args[0] == "--child":
        child(views, slots)
        return
    for setting in args or [""]:
        env = dict(os.environ)
        for kv in setting.split():
            k, v = kv.split("=", 1)
            env[k] = v
        env["AB_TAG"] = setting
        subprocess.run([sys.executable, __file__, "--views", str(views), "--slots", str(slots), "--child"],
                       env=env, check=False)


if __name__ == "__main__":
    main()
