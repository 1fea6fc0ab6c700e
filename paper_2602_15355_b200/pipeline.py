"""Host orchestration of one scoring pass (Alg. 1 L147-154 body): for every
candidate view, K1 project -> K2..K5 bin+sort -> K6 composite -> K7 score,
batched by view; then K8 top-k.  All arithmetic runs in libgsr's kernels;
this file only sizes buffers and sequences the C-ABI calls.

Batches alternate between ``n_slots`` independent slots, each with its own
CUDA stream, gsr context (scratch) and pipeline buffers, so the GPU runs
batch b's compositing (FP32-issue bound) concurrently with batch b+1's
projection and sorts (memory / latency bound): the two kinds of kernels
share the SMs instead of idling them in turn.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import gsr
from .gsr import Context, Gaussians, GsrError


CACHE_TAU, CACHE_BASE_BINS, CACHE_HOT_BINS = 0.6, 8, 16


def cache_bins(field: Gaussians, tile_start, tau: float = CACHE_TAU, ctx: Optional[Context] = None) -> np.ndarray:
    """NEXT-2b cache policy (§3.5, tau = 0.6 of §3.6):
    a tile whose mean per-Gaussian uncertainty exceeds tau keeps 16 cached
    orderings, the others 8 (gsr_order_cache_bins: one kernel, one readback)."""
    ctx = ctx or Context(field.planes.device.index or 0)
    return gsr.gsr_order_cache_bins(ctx, field, tile_start, tau, CACHE_BASE_BINS, CACHE_HOT_BINS)


def tiles_per_view(cam) -> int:
    W, H = int(cam["width"]), int(cam["height"])
    return ((W + 15) // 16) * ((H + 15) // 16)


@dataclass
class BatchOut:
    n_keys: int
    images: Optional[torch.Tensor] = None  # [V][H][W][4]


class _Slot:
    """One batch pipeline: K1..K5 on one stream (`stream`), K6/K7 on a
    higher-priority stream (`comp`) that waits for the sort; the next use of
    the slot waits for the previous composite.  With two slots the block
    scheduler fills the SMs the composite leaves free (its tail, ragged
    tiles) with the next batch's (latency-bound) sort kernels."""

    def __init__(self, dev, V: int, n: int, stream, comp=None):
        self.ctx = Context(dev.index or 0)
        self.stream = stream
        self.comp = comp if comp is not None else stream
        with torch.cuda.stream(stream):
            self.rec = torch.empty((V, max(n, 1), 12), dtype=torch.float32, device=dev)
            self.bin = torch.empty(10 * V * max(n, 1), dtype=torch.int32, device=dev)  # spans + depth + n_tiles
            self.n_frag = torch.zeros(2, dtype=torch.int64, device=dev)  # [blended, evaluated]
        self.capacity = 0
        self.vals = None
        self.keys = None
        self.ranges = None
        self.partial = None
        self.gray = None      # NEXT-4: [V][H][W] gray image of the batch
        self.partial2 = None  # NEXT-4: per-tile Sobel sums


class ViewScorer:
    """Scores candidate views of one Gaussian field on one GPU.

    ``batch_views`` views share one K1 launch (the parameter planes are read
    once per batch) and one pair of sorts.  Buffers grow on demand; the key
    capacity follows gsr_bin_sort's capacity protocol (GSR_ECAPACITY returns
    the required size; grow by 25 % and retry)."""

    def __init__(self, field: Gaussians, batch_views: int = 32, n_slots: int = 3, lod: Optional[gsr.Lod] = None,
                 order_tiles=None, composite_residency: Optional[int] = None):
        self.field = field
        self.lod = lod  # NEXT-2 LOD blending (opacity multiplier in K1), or None
        # NEXT-2b: (tile_start, bins, centres) -> cached view-direction orderings
        # replace the per-view depth sort (approximate blend order)
        self.dev = field.planes.device
        self.V = min(int(batch_views), gsr.GSR_MAX_VIEWS)
        self.slots: List[_Slot] = []
        lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
        for _ in range(max(1, n_slots)):
            if n_slots > 1:
                # composite stream high priority (measured: 2,910 views/s vs 2,904 with the sorts
                # high, and K6's event spans no longer include SMs lent to the sorts);
                # GSR_PRIO=sort / equal for the A/B
                ps, pc = {"sort": (hi, lo), "equal": (lo, lo)}.get(os.environ.get("GSR_PRIO", ""), (lo, hi))
                self.slots.append(_Slot(self.dev, self.V, field.n, torch.cuda.Stream(self.dev, priority=ps),
                                        torch.cuda.Stream(self.dev, priority=pc)))
            else:
                self.slots.append(_Slot(self.dev, self.V, field.n, torch.cuda.Stream(self.dev)))
        self.ctx = self.slots[0].ctx
        # K6 launch shape (gsr_set_composite_residency): 0 = one block per
        # strip; k > 0 = a persistent grid of k blocks per SM, so the next
        # batch's sort kernels co-run on the SMs' remaining room.  Workload-
        # dependent: c3 3,401 vs 3,336 views/s at k = 10 with
        # three slots, c2 10,014 vs 10,731 with two, c4 equal
        self.composite_residency = int(composite_residency or 0)
        for s_ in self.slots:
            s_.ctx.set_composite_residency(self.composite_residency)
        # diagnostic fragment counters (n_frag: blended fragments, evaluated
        # pairs), off by default: K6 then runs its variant without the per-hit
        # bookkeeping (c2: 3.5 % of the pass)
        self.count_fragments = False
        self.last_keys: List[int] = []
        self.order_cache = None
        if order_tiles is not None:
            self.order_cache = gsr.OrderCache(self.ctx, field, *order_tiles)
            torch.cuda.synchronize(self.dev)

    # ------------------------------------------------------------------ helpers
    @property
    def n_frag(self) -> torch.Tensor:
        """[blended fragments, evaluated pairs] summed over slots (device),
        accumulated by passes run with ``count_fragments = True``."""
        return torch.stack([s.n_frag for s in self.slots]).sum(0)

    def reset_counters(self):
        for s in self.slots:
            s.n_frag.zero_()

    def timing(self, enable: bool = True):
        for s in self.slots:
            s.ctx.timing(enable)

    def timing_read(self) -> dict:
        acc = None
        for s in self.slots:
            t = s.ctx.timing_read()
            if acc is None:
                acc = t
            else:
                for k, v in t.items():
                    for f in v:
                        acc[k][f] += v[f]
        return acc

    # Slot buffers are allocated with the slot's stream current, so the caching
    # allocator only recycles them in that stream's order (a replaced buffer may
    # still be read by the slot's previous, not yet finished, composite).
    @staticmethod
    def _ensure_keys(slot: _Slot, cap: int, want_keys: bool):
        if cap > slot.capacity or (want_keys and slot.keys is None):
            slot.capacity = max(cap, slot.capacity)
            with torch.cuda.stream(slot.stream):
                slot.vals = torch.empty(max(slot.capacity, 1), dtype=torch.int32, device=slot.rec.device)
                slot.keys = (torch.empty(max(slot.capacity, 1), dtype=torch.int64, device=slot.rec.device)
                             if want_keys else None)

    @staticmethod
    def _ensure_tiles(slot: _Slot, T: int):
        if slot.ranges is None or slot.ranges.shape[0] < T:
            with torch.cuda.stream(slot.stream):
                slot.ranges = torch.empty((T, 2), dtype=torch.int32, device=slot.rec.device)
                slot.partial = torch.empty(T, dtype=torch.float32, device=slot.rec.device)

    # ------------------------------------------------------------------ batches
    def run_batch(self, cams: np.ndarray, scores_out: torch.Tensor, images: Optional[torch.Tensor] = None,
                  t_final=None, n_contrib=None, want_keys: bool = False, slot: int = 0) -> BatchOut:
        """Score len(cams) <= batch_views same-resolution views into
        scores_out[0:len(cams)], enqueued on the slot's stream.  Standalone
        calls are ordered after, and joined back into, the caller's stream."""
        caller = torch.cuda.current_stream(self.dev)
        S = self.slots[slot]
        S.stream.wait_stream(caller)
        S.comp.wait_stream(caller)
        out = self._enqueue(S, cams, scores_out, images, t_final, n_contrib, want_keys)
        caller.wait_stream(S.comp)
        return out

    @staticmethod
    def _ensure_gray(slot: _Slot, V: int, H: int, W: int, T: int):
        if slot.gray is None or slot.gray.numel() < V * H * W:
            with torch.cuda.stream(slot.stream):
                slot.gray = torch.empty(V * H * W, dtype=torch.float32, device=slot.rec.device)
        if slot.partial2 is None or slot.partial2.numel() < T:
            with torch.cuda.stream(slot.stream):
                slot.partial2 = torch.empty(T, dtype=torch.float32, device=slot.rec.device)

    def _enqueue(self, S: _Slot, cams, scores_out, images=None, t_final=None, n_contrib=None,
                 want_keys: bool = False, sobel_out=None) -> BatchOut:
        cams = gsr.cams_array(cams)
        V = len(cams)
        assert 0 < V <= self.V
        n = self.field.n
        self._ensure_tiles(S, V * tiles_per_view(cams[0]))
        if S.capacity == 0:
            self._ensure_keys(S, max(1 << 20, 4 * n * V), want_keys)
        elif want_keys:
            self._ensure_keys(S, S.capacity, True)
        st = S.stream
        if S.comp is not S.stream:
            st.wait_stream(S.comp)  # the previous composite of this slot still reads rec / vals / ranges
        # rec / bin hold [V][n][12] and [10 V n] for THIS batch's V, packed from the
        # start of the (batch_views-sized) buffers: the base pointers are passed.
        gsr.gsr_project(S.ctx, self.field, cams, S.rec, S.bin, st, lod=self.lod)
        while True:
            try:
                if self.order_cache is not None:
                    K = gsr.gsr_bin_sort_cached(S.ctx, S.bin, n, cams, self.order_cache, S.vals, S.capacity,
                                                S.ranges, keys=S.keys if want_keys else None, stream=st)
                else:
                    K = gsr.gsr_bin_sort(S.ctx, S.bin, n, cams, S.vals, S.capacity, S.ranges,
                                         keys=S.keys if want_keys else None, stream=st)
                break
            except GsrError as e:
                if e.status != gsr.GSR_ECAPACITY:
                    raise
                self._ensure_keys(S, int(math.ceil(e.required * 1.25)) + 1024, want_keys)
        cs = S.comp
        if cs is not st:
            cs.wait_stream(st)
        gray = None
        if sobel_out is not None:
            W, H = int(cams[0]["width"]), int(cams[0]["height"])
            self._ensure_gray(S, V, H, W, V * tiles_per_view(cams[0]))
            gray = S.gray
        gsr.gsr_composite(S.ctx, S.rec, n, S.vals, S.ranges, cams, S.partial, rgbu=images, t_final=t_final,
                          n_contrib=n_contrib,
                          n_frag=S.n_frag if self.count_fragments else None, gray=gray, stream=cs)
        gsr.gsr_score_views(S.ctx, S.partial, cams, scores_out, cs)
        if sobel_out is not None:
            gsr.gsr_sobel_scores(S.ctx, gray, cams, S.partial2, sobel_out, cs)
        return BatchOut(K, images)

    def score_views(self, cams: np.ndarray, scores_out: Optional[torch.Tensor] = None,
                    sobel_out: Optional[torch.Tensor] = None,
                    images_out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Scores for all of ``cams`` (any count; same resolution), batches
        alternating over the slots' streams; the result is ordered back onto
        the caller's current stream.  ``sobel_out`` (optional [len(cams)]
        float tensor) also receives the NEXT-4 image term (mean Sobel
        gradient magnitude of each rendered view, PAPER.md eq:uncert_img);
        ``images_out`` (optional [len(cams)][H][W][4] float tensor) the
        composited (r, g, b, U) maps of every view."""
        cams = gsr.cams_array(cams)
        if scores_out is None:
            scores_out = torch.empty(len(cams), dtype=torch.float32, device=self.dev)
        caller = torch.cuda.current_stream(self.dev)
        for s in self.slots:
            s.stream.wait_stream(caller)  # inputs (field, scores_out) produced on the caller's stream
            s.comp.wait_stream(caller)
        self.last_keys = []
        for i, b0 in enumerate(range(0, len(cams), self.V)):
            b1 = min(len(cams), b0 + self.V)
            out = self._enqueue(self.slots[i % len(self.slots)], cams[b0:b1], scores_out[b0:b1],
                                images=None if images_out is None else images_out[b0:b1],
                                sobel_out=None if sobel_out is None else sobel_out[b0:b1])
            self.last_keys.append(out.n_keys)
        for s in self.slots:
            caller.wait_stream(s.comp)
        return scores_out

    def select(self, scores: torch.Tensor, k: int = 1, exclude=None) -> torch.Tensor:
        out = torch.empty(k, dtype=torch.int32, device=self.dev)
        gsr.gsr_select_nbv(self.ctx, scores, k, out, exclude, torch.cuda.current_stream(self.dev))
        return out


class Renderer:
    """Forward images + NEXT-3 backward for one batch of views -- the
    building block of UPDATE_GS (Alg. 1): ``forward(cams)``
    renders (r, g, b, U) images and keeps the batch's products;
    ``backward(dl_drgbu)`` adds dL/dparams (field plane layout) for an
    upstream image gradient.  All arithmetic is in libgsr's kernels."""

    def __init__(self, field: Gaussians, lod: Optional[gsr.Lod] = None):
        self.field = field
        self.lod = lod
        self.ctx = Context(field.planes.device.index or 0)
        self.dev = field.planes.device
        self._cams = None

    def forward(self, cams, stream=None) -> torch.Tensor:
        cams = gsr.cams_array(cams)
        V, n = len(cams), self.field.n
        W, H = int(cams[0]["width"]), int(cams[0]["height"])
        T = V * tiles_per_view(cams[0])
        # buffers are reused while the batch shape stays the same (a caller
        # holding the previous image must copy it first)
        shape = (V, n, W, H)
        if getattr(self, "_shape", None) != shape:
            self.rec = torch.empty((V, max(n, 1), 12), dtype=torch.float32, device=self.dev)
            self.bin = torch.empty(10 * V * max(n, 1), dtype=torch.int32, device=self.dev)
            self.ranges = torch.empty((T, 2), dtype=torch.int32, device=self.dev)
            self.partial = torch.empty(T, dtype=torch.float32, device=self.dev)
            self.rgbu = torch.empty((V, H, W, 4), dtype=torch.float32, device=self.dev)
            self._shape = shape
        gsr.gsr_project(self.ctx, self.field, cams, self.rec, self.bin, stream, lod=self.lod)
        cap = getattr(self, "_cap", 1 << 20)
        while True:
            if getattr(self, "vals", None) is None or self.vals.numel() < cap:
                self.vals = torch.empty(cap, dtype=torch.int32, device=self.dev)
            try:
                gsr.gsr_bin_sort(self.ctx, self.bin, n, cams, self.vals, cap, self.ranges, stream=stream)
                break
            except GsrError as e:
                if e.status != gsr.GSR_ECAPACITY:
                    raise
                cap = int(math.ceil(e.required * 1.25)) + 1024
        self._cap = cap
        gsr.gsr_composite(self.ctx, self.rec, n, self.vals, self.ranges, cams, self.partial, rgbu=self.rgbu,
                          stream=stream)
        self._cams = cams
        return self.rgbu

    def backward(self, dl_drgbu: torch.Tensor, grads: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        assert self._cams is not None, "forward() first"
        if grads is None:
            grads = torch.zeros_like(self.field.planes)
        gsr.gsr_backward(self.ctx, self.field, self._cams, self.rec, self.bin, self.vals, self.ranges, self.rgbu,
                         dl_drgbu.contiguous(), grads, lod=self.lod, stream=stream)
        return grads


class Refiner:
    """NEXT-3 UPDATE_GS refinement (Alg. 1, "bounded refinement
    (5k iterations per inserted image)", §4.1): per step, render the
    captured poses (Renderer.forward), the L2 photometric loss gradient
    against the captures, the backward rasterizer, and one projected Adam
    step on the field's planes -- all in libgsr kernels.  ``lr`` is a
    learning rate per (plane, component); the field is updated in place."""

    def __init__(self, field: Gaussians, lr, weights=(1.0, 1.0, 1.0, 0.0), lod: Optional[gsr.Lod] = None,
                 betas=(0.9, 0.999), eps: float = 1e-8):
        self.field = field
        self.renderer = Renderer(field, lod)
        self.lr = np.asarray(lr, dtype=np.float32).reshape(field.planes.shape[0], 4)
        self.weights = np.asarray(weights, dtype=np.float32)
        self.m = torch.zeros_like(field.planes)
        self.v = torch.zeros_like(field.planes)
        self.grads = torch.zeros_like(field.planes)
        self.betas, self.eps, self.t = betas, eps, 0
        self.loss = torch.zeros(1, dtype=torch.float64, device=field.planes.device)

    def step(self, cams, targets: torch.Tensor) -> torch.Tensor:
        """One refinement iteration on the poses ``cams`` (<= 64, one
        resolution) with capture images ``targets`` [V][H][W][4]; returns the
        pre-update loss (device scalar)."""
        img = self.renderer.forward(cams)
        dl = torch.empty_like(img)
        ctx = self.renderer.ctx
        gsr.gsr_l2_loss(ctx, img, targets.contiguous(), self.weights, dl_dimg=dl, loss=self.loss)
        self.grads.zero_()
        self.renderer.backward(dl, self.grads)
        self.t += 1
        gsr.gsr_adam_step(ctx, self.field.planes, self.grads, self.m, self.v, self.lr, self.t,
                          self.betas[0], self.betas[1], self.eps)
        return self.loss
