#!/usr/bin/env python
"""bench.py -- candidate views scored / s (+ fragments / s, roofline) for the
active-view scoring hot path of DAV-GSWT (arXiv 2602.15355) on B200.

Workload (BASELINE.json configs[2], the configuration the metric's target is
quoted on; fits one GPU): 1,000,000 Gaussians (SH degree 3), 1,024 candidate
cameras on a Fibonacci hemisphere of radius 4, 800x800 px, f = 900 px.
One step = one Alg. 1 scoring iteration: [N>1: broadcast
of the field] -> every candidate view projected, binned, sorted, composited
and scored (views sharded v mod N over ranks) -> [N>1: all-gather of the
scores] -> NBV selection.  Strong scaling: the 1,024 views are split over N.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gsr|reference]

N > 1 is launched by torchrun (one rank per GPU, NCCL).  Rank 0 prints ONE
JSON line.  `--impl reference` times the CPU oracle (the reference arm of
this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate_views_scored_per_sec"
UNIT = "views/s"
CONFIG_ID = 3


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="gsr", choices=["gsr", "reference"])
    p.add_argument("--batch-views", type=int, default=32)  # r2k: 32 3,547 / 48 3,546 / 64 3,518 views/s
    p.add_argument("--slots", type=int, default=3,
                   help="concurrent batch pipelines (stream pairs); r2k: 3: 3,547, 2: 3,443, 4: 3,542 views/s")
    p.add_argument("--k6-residency", type=int, default=10,
                   help="persistent K6 blocks per SM when batches overlap (gsr_set_composite_residency); r2k: 10: 3,547, 8: 3,535, 12: 3,512 views/s")
    p.add_argument("--cpu-views", type=int, default=0, help="oracle sample size (0 = auto)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the NEXT-1/2/4 extra measurements")
    return p.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return dict(hbm_gbs=float(d["hbm_gbs"]), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)), source="measured")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, source="fallback")


def load_traffic():
    """DRAM bytes (read + write) per launch of the roofline kernels, from the
    committed ncu --set full capture (profiles/traffic.json), or {}."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    return json.load(open(path)) if os.path.exists(path) else {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 8]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def cpu_model() -> str:
    """The host CPU's model name (/proc/cpuinfo), for the CPU baselines."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, scene, cfg_json):
    import oracle
    n_threads = os.cpu_count() or 1
    # one view per host thread per step (~16 s of wall time on the GPU box), so
    # the whole --steps K --warmup W run stays within a few minutes
    nv = args.cpu_views or max(4, min(32, n_threads))
    idx = np.linspace(0, len(scene.cameras) - 1, nv).round().astype(np.int64)
    cams = np.ascontiguousarray(scene.cameras[idx])
    oracle.build()
    times = []
    fr = 0
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        scores, nf, nk, _ = oracle.render_views(scene.field, cams, n_threads=n_threads)
        sel = oracle.select_topk(scores, 1)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
            fr = int(nf.sum())
        if step == 0 and args.warmup + args.steps > 2 and dt > 60:
            break
    t = float(np.mean(times)) if times else float("nan")
    v = nv / t
    sample = (f"{nv} strided views of the 1,024 (full O1-O6 oracle per view: projection, "
              f"duplication, qsort, tiled compositing, score) + top-1")
    return {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": 0,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg_json,
            "fragments_per_sec": fr / t,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": n_threads, "cpu_model": cpu_model(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cpu_baseline(scene, n_views: int):
    import oracle
    n_threads = os.cpu_count() or 1
    nv = n_views or max(4, min(32, n_threads))
    idx = np.linspace(0, len(scene.cameras) - 1, nv).round().astype(np.int64)
    cams = np.ascontiguousarray(scene.cameras[idx])
    oracle.build()
    t0 = time.perf_counter()
    scores, nf, nk, _ = oracle.render_views(scene.field, cams, n_threads=n_threads)
    dt = time.perf_counter() - t0
    return {"value": nv / dt, "unit": UNIT, "cores": n_threads, "cpu_model": cpu_model(), "kind": "oracle",
            "sample": f"{nv} strided views of the 1,024 at 800x800 (1M Gaussians), full O1-O6 oracle, "
                      f"{dt:.1f} s wall on {n_threads} threads", "fragments_per_sec": float(nf.sum()) / dt}


def bench_w2(gsr, dev, peaks, reps: int = 20):
    """NEXT-1: W2 latent scoring of N = 1000 candidates (M = 5, C = 4, 64 x 64;
    PAPER.md L135, L181), HBM roofline on the 2 M C H W floats read per view."""
    import torch
    import synth
    mu, s2 = synth.gen_latent_ensembles(1000, 5, 4, 64, 64, seed=0)
    m, s = torch.from_numpy(mu).to(dev), torch.from_numpy(s2).to(dev)
    sc = torch.empty(1000, device=dev)
    ctx = gsr.Context(dev.index or 0)
    for _ in range(3):
        gsr.gsr_w2_scores(ctx, m, s, sc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gsr.gsr_w2_scores(ctx, m, s, sc)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    byts = 2.0 * mu.nbytes
    return {"metric": "w2_candidates_scored_per_sec", "value": round(1000 / t, 1), "unit": "views/s",
            "ms_per_pass": round(t * 1e3, 4), "config": "N=1000, M=5, C=4, 64x64 (synthetic latents)",
            "roofline": {"bound": "hbm", "achieved": round(byts / t / 1e9, 1), "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": round(byts / t / 1e9 / peaks["hbm_gbs"], 4)}}


def bench_sobel(gsr, dev, peaks, reps: int = 20):
    """NEXT-4: Sobel image term (PAPER.md eq:uncert_img) over the gray images of
    one 32-view c3 batch (800 x 800, the scoring pass's batch size), HBM
    roofline on the 4 B read per pixel (the two halo rows per 16-row band hit
    L2) + 8 B per tile partial."""
    import torch
    import synth
    V, W, H = 32, 800, 800
    g = torch.rand((V, H, W), device=dev)
    cams = synth.fibonacci_cameras(V, 4.0, W, H, 900.0)
    tpv = ((W + 15) // 16) * ((H + 15) // 16)
    part = torch.empty(V * tpv, device=dev)
    sc = torch.empty(V, device=dev)
    ctx = gsr.Context(dev.index or 0)
    for _ in range(3):
        gsr.gsr_sobel_scores(ctx, g, cams, part, sc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gsr.gsr_sobel_scores(ctx, g, cams, part, sc)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    byts = 4.0 * V * W * H + 8.0 * V * tpv
    return {"metric": "sobel_views_scored_per_sec", "value": round(V / t, 1), "unit": "views/s",
            "ms_per_batch": round(t * 1e3, 4), "config": "32 views x 800x800 gray (c3 resolution, the scoring pass's batch)",
            "roofline": {"bound": "hbm", "achieved": round(byts / t / 1e9, 1), "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": round(byts / t / 1e9 / peaks["hbm_gbs"], 4)}}


def bench_wang(dev, steps: int = 3):
    """NEXT-2 on the config-4 fly-over (64 views, 1920x1080, the 4x4 Wang
    assembly): (a) LOD blending (PAPER.md eq:lod_blend) -- six levels per tile
    (10.7 M Gaussians; K1 scales opacities by the level weights and culls the
    inactive levels) vs the level-0-only assembly (8 M, configs[3]); (b) the
    uncertainty-guided cached view-direction orderings (§3.5) replacing
    the per-view depth sort, with the mean relative score change vs exact."""
    import torch
    import synth
    from paper_2602_15355_b200 import Gaussians, Lod
    from paper_2602_15355_b200.pipeline import ViewScorer, cache_bins
    cams = synth.flyover_cameras(64, 1920, 1080, 1500.0)
    out = {"config": "c4 fly-over 64 views 1920x1080; LOD: 6 levels/tile (1/4 count, 2.3x scale per level), "
                      "D = 1.5, 3, 6, 12, 24, delta = 0.25; cache: 8/16 azimuthal bins per tile (tau = 0.6)"}

    def run(G, L, tiles):
        sc = ViewScorer(G, batch_views=16, n_slots=2, lod=L, order_tiles=tiles)
        for _ in range(2):
            s = sc.score_views(cams)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            s = sc.score_views(cams)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / steps / 1e3
        return {"gaussians": G.n, "views_per_sec": round(64 / t, 1), "ms_per_pass": round(t * 1e3, 2),
                "keys_per_view": int(sum(sc.last_keys) / 64)}, s

    for name, lod in (("level0_only", False), ("lod", True)):
        if lod:
            fld, ld = synth.gen_config4_lod(500_000)
        else:
            fld, ld = synth.gen_config4_field(500_000), None
        start, centres = synth.config4_tiles(500_000, lod=lod)
        G = Gaussians(torch.from_numpy(fld.planes).to(dev), fld.sh_degree)
        del fld
        L = None if ld is None else Lod(torch.from_numpy(ld.tile_level).to(dev), ld.levels, ld.delta, ld.thresholds)
        exact, s_exact = run(G, L, None)
        bins = cache_bins(G, start)
        cached, s_cached = run(G, L, (start, bins, centres))
        cached["bins"] = sorted(set(int(b) for b in bins))
        cached["mean_rel_score_change_vs_exact"] = float(((s_cached - s_exact).abs() / s_exact).mean().item())
        out[name] = {"exact_sort": exact, "cached_order": cached}
        del G, L
        torch.cuda.empty_cache()
    return out


def bench_backward(G, dev, reps: int = 3):
    """NEXT-3: forward images + backward rasterizer for one 16-view c3 batch
    (1 M Gaussians, 800x800), upstream gradient of an L2 photometric loss
    against a perturbed copy of the image; device time per view."""
    import torch
    import synth
    from paper_2602_15355_b200.pipeline import Renderer
    cams = synth.fibonacci_cameras(1024, 4.0, 800, 800, 900.0)[::64]
    r = Renderer(G)
    img = r.forward(cams)
    target = img + 0.01 * torch.randn_like(img)
    grads = torch.zeros_like(G.planes)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    fw = bw = 0.0
    for i in range(reps + 1):
        e[0].record()
        img = r.forward(cams)
        e[1].record()
        r.backward(2.0 * (img - target), grads)
        e[2].record()
        torch.cuda.synchronize()
        if i:
            fw += e[0].elapsed_time(e[1])
            bw += e[1].elapsed_time(e[2])
    fw, bw = fw / reps, bw / reps
    # K6b / K1b device times (their own stages) and K6b's FP32 roofline: the
    # walk's evaluated pairs E and blended fragments F from one counted,
    # untimed composite of the same batch; work = 28 E (the forward's walk) +
    # 56 F (per blended pair: the forward blend 8, 1 / (1 - alpha) 2, dL/dalpha
    # over four channels 24, dL/dpower and the ten parameter gradients 22)
    from paper_2602_15355_b200 import gsr
    nf = torch.zeros(2, dtype=torch.int64, device=dev)
    gsr.gsr_composite(r.ctx, r.rec, G.n, r.vals, r.ranges, cams, r.partial, n_frag=nf)
    torch.cuda.synchronize()
    E, F = float(nf[1].item()), float(nf[0].item())
    r.ctx.timing(True)
    r.ctx.timing_read()
    for _ in range(reps):
        r.backward(2.0 * (img - target), grads)
    st = r.ctx.timing_read()
    r.ctx.timing(False)
    k6b_ms, k1b_ms = st["backward"]["ms"] / reps, st["backward_project"]["ms"] / reps
    peak_ops = 148 * 128 * 1965e6 / 1e12
    k6b_ops = (28.0 * E + 56.0 * F) / (k6b_ms / 1e3) / 1e12
    k1b_gbs = st["backward_project"]["bytes"] / reps / (k1b_ms / 1e3) / 1e9
    peaks = load_peaks()
    # one UPDATE_GS refinement iteration (render, L2 loss gradient, backward,
    # projected Adam) on a copy of the field against the perturbed captures
    from paper_2602_15355_b200 import Gaussians
    from paper_2602_15355_b200.pipeline import Refiner
    G2 = Gaussians(G.planes.clone(), G.sh_degree)
    lr = np.full((G2.planes.shape[0], 4), 1e-3, np.float32)
    ref = Refiner(G2, lr)
    ref.step(cams, target)
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(reps):
        ref.step(cams, target)
    e[1].record()
    torch.cuda.synchronize()
    it = e[0].elapsed_time(e[1]) / reps
    del ref, G2
    torch.cuda.empty_cache()
    return {"metric": "forward_backward_views_per_sec", "value": round(16 / ((fw + bw) / 1e3), 1), "unit": "views/s",
            "forward_ms_per_batch": round(fw, 3), "backward_ms_per_batch": round(bw, 3),
            "refine_iterations_per_sec": round(1e3 / it, 1), "refine_ms_per_iteration": round(it, 3),
            "k6b_ms_per_batch": round(k6b_ms, 3), "k1b_ms_per_batch": round(k1b_ms, 3),
            "roofline": {"bound": "alu", "kernel": "k6_backward", "achieved": round(k6b_ops, 2),
                         "peak": round(peak_ops, 2), "unit": "Top/s", "frac": round(k6b_ops / peak_ops, 4),
                         "work": "28 FP32 ops per evaluated (pixel, entry) pair of the forward walk + 56 per "
                                 "blended fragment (gradient chain), per 16-view batch",
                         "peak_source": "148 SMs x 128 FP32 lanes x 1965 MHz (max SM clock)"},
            "roofline_k1b": {"bound": "hbm", "kernel": "k1_backward", "achieved": round(k1b_gbs, 1),
                             "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(k1b_gbs / peaks["hbm_gbs"], 4),
                             "work": "40 B per visible pair + 4 B per (view, g) + 2 x 16 B per plane per Gaussian "
                                     "(ALU-heavy: the chain rule per (view, g) at SH degree 3)"},
            "config": "c3 field (1M Gaussians, SH 3), 16 views 800x800, L2 loss vs a perturbed image; "
                      "refinement iteration = forward + loss gradient + backward + Adam on 16 views"}


def bench_hierarchical(dev, reps: int = 2):
    """configs[4] (hierarchical coarse-to-fine scoring, PAPER.md L5 / Alg. 1
    top-k): 2 M Gaussians; coarse pass over 4,096 candidates at 256x256
    (f = 288), top-64 by (score desc, index asc), fine pass re-rendering those
    64 at 1024x1024 (f = 1152), NBV = fine argmax.  One GPU (the all-gather
    between the passes is the N > 1 plumbing of distributed.hierarchical_select)."""
    import torch
    import synth
    from paper_2602_15355_b200 import Gaussians
    from paper_2602_15355_b200.distributed import hierarchical_select
    from paper_2602_15355_b200.pipeline import ViewScorer
    sc = synth.make_scene(5)
    G = Gaussians(torch.from_numpy(sc.field.planes).to(dev), sc.field.sh_degree)
    coarse = ViewScorer(G, batch_views=32, n_slots=2)  # measured: 32 > 64 > 16 views per batch at 256^2
    fine = ViewScorer(G, batch_views=16, n_slots=2)

    def run():
        return hierarchical_select(sc.cameras, lambda c: synth.with_resolution(c, 1024, 1024, 1152.0),
                                   coarse.score_views, fine.score_views,
                                   lambda s, k, ex: coarse.select(s, k, ex), top_k=64)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        cs, top, fs, nbv = run()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    return {"metric": "hierarchical_passes_per_sec", "value": round(1.0 / t, 2), "unit": "passes/s",
            "ms_per_pass": round(t * 1e3, 2), "candidate_views_per_sec": round((4096 + 64) / t, 1),
            "nbv": int(nbv), "config": "c5: 2M Gaussians, 4096 coarse views 256^2 -> top-64 fine 1024^2"}


def bench_configs(dev, steps: int = 3):
    """Views/s of every BASELINE.json config on one GPU (the headline line is
    configs[2]; configs[3] and [4] also appear in next2_wang /
    c5_hierarchical): c1 10k / 16 views 128^2, c2 200k terrain / 256 views
    512^2, c4 8M Wang assembly / 64 fly-over views 1920x1080."""
    import torch
    import synth
    from paper_2602_15355_b200 import Gaussians
    from paper_2602_15355_b200.pipeline import ViewScorer
    out = {}
    for cfg in (1, 2, 4):
        sc = synth.make_scene(cfg)
        G = Gaussians(torch.from_numpy(sc.field.planes).to(dev), sc.field.sh_degree)
        s = ViewScorer(G, batch_views=16, n_slots=2)
        nv = len(sc.cameras)
        s.count_fragments = True  # one counted pass, untimed
        s.reset_counters()
        s.score_views(sc.cameras)
        torch.cuda.synchronize()
        fr = float(s.n_frag[0].item())
        s.count_fragments = False
        s.score_views(sc.cameras)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            s.score_views(sc.cameras)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / steps / 1e3
        out[synth.CONFIG_NAMES[cfg]] = {"views_per_sec": round(nv / t, 1), "ms_per_pass": round(t * 1e3, 2),
                                        "fragments_per_sec": round(fr / t, 1),
                                        "keys_per_view": int(sum(s.last_keys) / nv)}
        del s, G, sc
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import synth
    cfg_json = {"workload": synth.CONFIG_NAMES[CONFIG_ID], "gaussians": 1_000_000, "sh_degree": 3,
                "views": 1024, "width": 800, "height": 800, "focal_px": 900, "tile": 16,
                "batch_views": args.batch_views, "streams": args.slots,
                "parallelism": f"dp{world} (views v mod N)",
                "l2": f"inputs larger than L2: 240 MB field + ~{0.055 * args.batch_views:.1f} GB keys per "
                      f"{args.batch_views}-view batch, no flush"}

    if args.impl == "reference":
        if rank != 0:
            return
        scene = synth.make_scene(CONFIG_ID)
        print(json.dumps(run_reference(args, scene, cfg_json)), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2602_15355_b200 import Gaussians, gsr
    from paper_2602_15355_b200.distributed import broadcast_field, score_and_select
    from paper_2602_15355_b200.pipeline import ViewScorer

    # GSR_BENCH_BACKEND=gloo: functional check of the N > 1 code path on a box
    # with fewer GPUs than ranks (ranks share devices; host-mediated
    # collectives; its timings are not scaling numbers)
    backend = os.environ.get("GSR_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    scene = synth.make_scene(CONFIG_ID) if rank == 0 else synth.make_scene(CONFIG_ID, n_override=1, views=1024)
    P = 3 + synth.n_sh_planes(3)
    n = 1_000_000
    host_planes = torch.empty((P, n, 4), dtype=torch.float32).pin_memory()
    if rank == 0:
        host_planes.copy_(torch.from_numpy(scene.field.planes))
    cams = synth.fibonacci_cameras(1024, 4.0, 800, 800, 900.0)
    planes = torch.empty((P, n, 4), dtype=torch.float32, device=dev)
    planes.copy_(host_planes, non_blocking=False)
    G = Gaussians(planes, 3)
    # K6 as a persistent grid of 10 blocks per SM beside the next batch's sorts
    # when batches overlap (c3 3,401 vs 3,336 views/s)
    scorer = ViewScorer(G, batch_views=args.batch_views, n_slots=args.slots,
                        composite_residency=args.k6_residency if args.slots > 1 else 0)

    def score_fn(c):
        return scorer.score_views(c)

    def select_fn(scores, k, exclude):
        return scorer.select(scores, k, exclude)

    # e2e result staging (page-locked, so the C-ABI copies are asynchronous)
    host_scores = torch.empty(1024, dtype=torch.float32).pin_memory()
    host_sel = torch.empty(1, dtype=torch.int32).pin_memory()

    def step(e2e: bool = False):
        if e2e and rank == 0:
            # H2D of the step's inputs through the C ABI (gsr_upload, pinned host planes)
            gsr.gsr_upload(scorer.ctx, planes, host_planes)
        broadcast_field(planes)
        scores, sel = score_and_select(cams, score_fn, select_fn, 1)
        if e2e:
            # D2H of the step's result through the C ABI (gsr_download), read on the host
            gsr.gsr_download(scorer.ctx, host_scores, scores)
            gsr.gsr_download(scorer.ctx, host_sel, sel)
            torch.cuda.current_stream().synchronize()
            return host_sel
        return sel

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def count_step():
        """The fragment counters of one step (untimed; they depend only on the
        workload, which every step repeats): the timed steps run K6 without
        the counting bookkeeping."""
        scorer.count_fragments = True
        scorer.reset_counters()
        step()
        barrier()
        fr = scorer.n_frag.clone().to(torch.float64)
        scorer.count_fragments = False
        if world > 1:
            dist.all_reduce(fr, op=dist.ReduceOp.SUM)
        return fr.tolist()

    def timed(k, e2e=False, stage_timing=False):
        scorer.timing(stage_timing)
        scorer.timing_read()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        for _ in range(k):
            step(e2e)
        ev1.record()
        barrier()
        wall = time.perf_counter() - t0
        ms = ev0.elapsed_time(ev1)
        stages = scorer.timing_read()
        scorer.timing(False)
        t = torch.tensor([ms, wall * 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0].item()), float(t[1].item()), [c * k for c in counts], stages

    counts = count_step()
    for _ in range(args.warmup):
        step()
    barrier()

    clocks = ClockSampler(local)
    clocks.start()
    ms, wall_ms, frags, stages = timed(args.steps, stage_timing=True)
    clk = clocks.stop()
    # value: whole-job views/s, device time max over ranks
    views_per_s = 1024 * args.steps / (ms / 1e3)
    frag_per_s = frags[0] / (ms / 1e3)
    eval_per_s = frags[1] / (ms / 1e3)

    # e2e: through the public API with the field copied H2D from pinned host
    # memory every step and the scores + NBV read back D2H, both copies
    # through the C ABI (gsr_upload / gsr_download)
    e2e = None
    if not args.no_e2e:
        ms_e, _, _, _ = timed(args.steps, e2e=True)
        e2e = {"value": 1024 * args.steps / (ms_e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(planes.numel() * 4 + 96 * 1024),
               "d2h_bytes_per_step": int(4 * 1024 + 4)}

    peaks = load_peaks()
    st_ms = {k: v["ms"] / args.steps for k, v in stages.items()}
    st_by = {k: v["bytes"] / args.steps for k, v in stages.items()}
    launches = sum(v["launches"] for v in stages.values())
    stage_tab = {k: {"ms_per_step": round(st_ms[k], 4), "algo_GB_per_step": round(st_by[k] / 1e9, 4),
                     "GB_per_s": round(st_by[k] / (st_ms[k] / 1e3) / 1e9, 1) if st_ms[k] > 0 else None,
                     "launches_per_step": stages[k]["launches"] / args.steps}
                 for k in stages if stages[k]["launches"]}
    # Rooflines: the dominant kernel of the step is
    # K6 (composite), bound by FP32/ALU issue; its algorithmic work is SURVEY
    # §8(d)'s 28 ops per evaluated (pixel, entry) pair of the plain definition +
    # 8 per blended fragment.  The key sort (K4c tile sort) is reported against
    # HBM, as the north_star asks.  Both use device times from CUDA events
    # bracketing those kernels on their launch stream inside the timed region.
    f_clk = (clk.get("sm_mhz") or peaks["sm_max_mhz"]) * 1e6
    peak_ops = 148 * 128 * f_clk / 1e12  # FP32 lanes x clock, Top/s
    traffic = load_traffic()
    if traffic.get("views_per_launch") not in (None, args.batch_views):
        traffic = {}  # the committed capture was taken at another batch size: no per-launch figure
    comp_ops = (28.0 * frags[1] + 8.0 * frags[0]) / args.steps  # per step
    comp_t = st_ms["composite"] / 1e3
    ach_ops = comp_ops / comp_t / 1e12
    n_comp = max(1, stages["composite"]["launches"] // args.steps)
    roof = {"bound": "alu", "kernel": "k6_composite", "achieved": round(ach_ops, 2), "peak": round(peak_ops, 2),
            "unit": "Top/s", "frac": round(ach_ops / peak_ops, 4),
            "traffic": traffic.get("k6_composite"),
            "ncu": traffic.get("k6_ncu"),  # FP32-pipe and shared-memory fractions (north_star), committed capture
            "work": "28 FP32 ops per (pixel, list entry) pair the plain definition evaluates + 8 per blended "
                    f"fragment, per launch = {args.batch_views} views",
            "peak_source": f"148 SMs x 128 FP32 lanes x {f_clk / 1e6:.0f} MHz (median SM clock under load)",
            "note": "SURVEY.md §8 L292-306 work model: the culled kernel skips most of the plain definition's "
                    "pairs and runs its hit loop in packed FP32, so this throughput of plain-definition work can "
                    "exceed the lane peak alone on the GPU (roofline_isolated); pipe utilisation is ncu.fma_pipe_pct. "
                    "In the pipeline K6 runs as a persistent grid of 10 blocks per SM beside the next batch's sort "
                    "kernels, so its launch spans include SM time the sorts use",
            # its event spans / the device step time (stage spans of the two
            # slots overlap, so they do not add up to the step)
            "share_of_step": round(st_ms["composite"] / (ms / args.steps), 3),
            "launches_per_step": n_comp}
    if traffic.get("k6_ncu", {}).get("warp_inst") and frags[1] > 0:
        # lane-instructions K6 issues per evaluated (pixel, entry) pair
        roof["lane_inst_per_eval_pair"] = round(
            traffic["k6_ncu"]["warp_inst"] * 32 / (frags[1] / max(1, n_comp // 2 * args.steps)), 2)
    ach_sort = st_by["tile_sort"] / (st_ms["tile_sort"] / 1e3) / 1e9
    roof_sort = {"bound": "hbm", "kernel": "tile_sort (K4c counting scatter: chunk histograms + column scan + "
                                            "ranked scatter)", "achieved": round(ach_sort, 1),
                 "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach_sort / peaks["hbm_gbs"], 4),
                 "traffic": traffic.get("tile_sort"),
                 "peak_source": peaks["source"] + " hbm_gbs (MEASURED_PEAKS.json)",
                 "share_of_step": round(st_ms["tile_sort"] / (ms / args.steps), 3)}

    # the same K6 roofline with K6 alone on the GPU (one slot, one step): the
    # two-stream spans above include time the composite shares with the sorts
    iso = iso_sort = iso_stages = with_maps = None
    if not args.no_extras and world == 1:
        iso_scorer = ViewScorer(G, batch_views=args.batch_views, n_slots=1)
        iso_scorer.reset_counters()
        iso_scorer.count_fragments = True
        iso_scorer.score_views(cams)  # counted, untimed
        torch.cuda.synchronize()
        ifr = iso_scorer.n_frag.to(torch.float64).tolist()
        iso_scorer.count_fragments = False
        iso_scorer.timing(True)
        iso_scorer.timing_read()
        torch.cuda.synchronize()
        iso_scorer.score_views(cams)
        torch.cuda.synchronize()
        ist = iso_scorer.timing_read()
        it = ist["composite"]["ms"] / 1e3
        iso_ops = (28.0 * ifr[1] + 8.0 * ifr[0]) / it / 1e12
        iso = {"bound": "alu", "kernel": "k6_composite (one stream)", "achieved": round(iso_ops, 2),
               "peak": round(peak_ops, 2), "unit": "Top/s", "frac": round(iso_ops / peak_ops, 4),
               "ms_per_step": round(ist["composite"]["ms"], 2),
               "share_of_serial_step": round(ist["composite"]["ms"] / sum(v["ms"] for v in ist.values()), 3)}
        # the key sort alone too (one stream: no SMs shared with a composite)
        iso_sort_gbs = ist["tile_sort"]["bytes"] / (ist["tile_sort"]["ms"] / 1e3) / 1e9
        iso_sort = {"bound": "hbm", "kernel": "tile_sort (one stream)", "achieved": round(iso_sort_gbs, 1),
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(iso_sort_gbs / peaks["hbm_gbs"], 4),
                    "ms_per_step": round(ist["tile_sort"]["ms"], 2),
                    "share_of_serial_step": round(ist["tile_sort"]["ms"] / sum(v["ms"] for v in ist.values()), 3)}
        # every stage alone on one stream (the kernels' own rates; inside the
        # pipeline a stage's event spans also hold time it waits for SMs)
        iso_stages = {k: {"ms_per_step": round(v["ms"], 3),
                          "algo_GB_per_step": round(v["bytes"] / 1e9, 3),
                          "GB_per_s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else None,
                          "frac_hbm": round(v["bytes"] / (v["ms"] / 1e3) / 1e9 / peaks["hbm_gbs"], 4)
                          if v["ms"] > 0 else None}
                      for k, v in ist.items() if v["launches"]}
        iso_scorer.timing(False)
        del iso_scorer
        torch.cuda.empty_cache()
        # the same step also writing every view's (r, g, b, U) map (north_star:
        # "with oracle-matching maps"): 1,024 x 800 x 800 x 16 B = 10.5 GB
        # written per step into one resident tensor
        maps = torch.empty((1024, 800, 800, 4), dtype=torch.float32, device=dev)
        sc_m = torch.empty(1024, dtype=torch.float32, device=dev)
        scorer.score_views(cams, sc_m, images_out=maps)
        barrier()
        em0, em1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        em0.record()
        for _ in range(args.steps):
            scorer.score_views(cams, sc_m, images_out=maps)
            scorer.select(sc_m, 1)
        em1.record()
        barrier()
        mms = em0.elapsed_time(em1) / args.steps
        with_maps = {"value": round(1024 / (mms / 1e3), 2), "unit": UNIT, "ms_per_step": round(mms, 3),
                     "maps_GB_per_step": round(maps.numel() * 4 / 1e9, 2),
                     "what": "the timed step with every view's RGBU map written to a resident [1024][800][800][4] "
                             "float tensor"}
        del maps
        torch.cuda.empty_cache()

    # the two collectives timed on their own (CUDA events on
    # the current stream, max over ranks): C1 broadcast of the 240 MB field
    # and C2 all-gather of the scores (both are inside every timed step above)
    coll = None
    if world > 1:
        from paper_2602_15355_b200.distributed import gather_scores
        reps = 5
        loc = torch.zeros((1024 + world - 1) // world, dtype=torch.float32, device=dev)
        barrier()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        for _ in range(reps):
            broadcast_field(planes)
        e1.record()
        for _ in range(reps):
            gather_scores(loc, 1024)
        e2.record()
        barrier()
        ct = torch.tensor([e0.elapsed_time(e1) / reps, e1.elapsed_time(e2) / reps], dtype=torch.float64,
                          device=dev)
        dist.all_reduce(ct, op=dist.ReduceOp.MAX)
        bms, gms = float(ct[0].item()), float(ct[1].item())
        coll = {"backend": backend, "broadcast_ms": round(bms, 4),
                "broadcast_GB_per_s": round(planes.numel() * 4 / (bms / 1e3) / 1e9, 1),
                "all_gather_ms": round(gms, 4), "bytes_broadcast": int(planes.numel() * 4)}

    line = {"metric": METRIC, "value": round(views_per_s, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator of BASELINE.json configs[2]; no dataset)",
            "config": cfg_json, "fragments_per_sec": frag_per_s, "evaluated_pairs_per_sec": eval_per_s,
            "wall_ms_per_step": round(wall_ms / args.steps, 3), "roofline": roof, "roofline_isolated": iso,
            # the key sort's own rate is the single-stream figure: inside the
            # pipeline its low-priority event spans also hold the time it waits
            # for SMs the composite holds (kept as roofline_sort_pipeline)
            "roofline_sort": iso_sort if iso_sort is not None else roof_sort,
            "roofline_sort_pipeline": roof_sort,
            "stages": stage_tab, "stages_single_stream": iso_stages, "with_maps": with_maps,
            "gpu_launches": int(launches * world), "clocks": clk, "e2e": e2e, "collectives": coll,
            "keys_per_step_rank0": int(sum(scorer.last_keys))}
    if rank == 0 and world == 1 and not args.no_extras:  # single-GPU extras (skipped in the scaling runs)
        line["next1_w2"] = bench_w2(gsr, dev, peaks)
        line["next4_sobel"] = bench_sobel(gsr, dev, peaks)
        line["next3_backward"] = bench_backward(G, dev)
        line["next2_wang"] = bench_wang(dev)
        line["c5_hierarchical"] = bench_hierarchical(dev)
        line["configs"] = bench_configs(dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(scene, args.cpu_views)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
