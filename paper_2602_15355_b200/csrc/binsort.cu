// binsort.cu -- K2..K5: tile-count scan, key duplication, onesweep radix
// sort, per-tile ranges (O2/O3).
//
// The (view, tile)-major, depth-minor order of the duplicated keys is produced
// in two levels, each a stable LSD onesweep radix sort with decoupled
// look-back (one upfront histogram, one scatter pass per 8-bit digit):
//
//   K2  k2_compact   single-pass look-back scan of n_tiles over (view, g):
//                    compacts the visible pairs into 64-bit depth keys
//                    (view << 32 | depth bits) + value g, counts K, and
//                    accumulates the digit histograms of the depth sort.
//   K4a onesweep     depth sort of the visible pairs (32 + log2 V bits).
//   K3  k3_emit      single-pass look-back scan of n_tiles in depth order,
//                    warp-cooperative load-balanced emission of the 32-bit
//                    (view*tiles + tile) keys, per-tile counts with
//                    warp-aggregated atomics (match_any + one atomicAdd).
//   K5  k5_ranges    per-tile [start, end) = exclusive scan of the counts,
//                    plus the digit histograms of the tile sort (from counts).
//   K4b onesweep     stable tile sort of the duplicated list (log2(V*tiles)
//                    bits = 2 passes for every config); the last pass writes the
//                    sorted values (and, if asked, the 64-bit keys).
//
// Because LSD radix sorting is stable and the emission order is already
// (view, depth, g), the result is exactly the (key, value) lexicographic order
// of the full 64-bit keys -- bit-identical to sorting the 64-bit keys
// directly (gsr_sort_pairs_u64, also exported), at a third of the HBM traffic.
#include "gsr_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

namespace gsr {
namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint64_t LB_AGG = 1ull << 62, LB_INC = 2ull << 62, LB_VAL = (1ull << 62) - 1;
constexpr uint32_t DG_AGG = 1u << 30, DG_INC = 2u << 30, DG_VAL = (1u << 30) - 1;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// Look-back words are read and written with volatile relaxed gpu-scope
// accesses: the flag and the count share one word, so no fence is needed, but
// the loads MUST be volatile -- with a plain (CSE-able) load the compiler may
// assume a spin on an unchanged word never happens and fold it away.
__device__ __forceinline__ uint32_t ld_word(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_word(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_word(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_word(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(FULL, v, o);
    if ((int)lane_id() >= o) v += t;
  }
  return v;
}

#ifndef SCAN_PTX
#define SCAN_PTX 1
#endif
#if SCAN_PTX
// u32: the shuffle's own in-range predicate guards the add (2 instructions per
// step instead of shuffle, select, add)
template <>
__device__ __forceinline__ uint32_t warp_incl_scan<uint32_t>(uint32_t v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
                 "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t@p add.u32 %0, %0, t;\n\t}"
                 : "+r"(v) : "r"(o));
  return v;
}
#endif

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Warp-parallel decoupled look-back over a chain of flagged 64-bit words.
// Called by a full warp for block `bid` > 0; returns the exclusive prefix.
__device__ uint64_t warp_lookback(const uint64_t* words, int64_t bid) {
  const uint32_t lane = lane_id();
  uint64_t excl = 0;
  int64_t base = bid - 1;
  while (true) {
    const int64_t idx = base - lane;
    uint64_t w = idx >= 0 ? ld_word(words + idx) : LB_INC;
    const uint32_t f = (uint32_t)(w >> 62);
    const uint32_t notready = __ballot_sync(FULL, f == 0);
    const uint32_t inc = __ballot_sync(FULL, f == 2);
    const uint32_t stop = notready | inc;
    if (stop == 0) {
      excl += warp_sum<uint64_t>(w & LB_VAL);
      base -= 32;
      continue;
    }
    const int first = __ffs(stop) - 1;
    const bool take = (int)lane < first || ((int)lane == first && (inc >> first & 1));
    excl += warp_sum<uint64_t>(take ? (w & LB_VAL) : 0);
    if (inc >> first & 1) break;
    base -= first;  // lanes before `first` were aggregates: consume and spin on `first`
  }
  return excl;
}

// Lanes whose bit b of d equals this lane's: the bit test, the ballot and the
// choice "ballot or its complement" as one PTX block, so ptxas loads several
// digit bits into predicates at once (R2P) and complements the ballots under
// predicates -- about 3 instructions per bit where the C++ form
// (bit ? bb : ~bb) kept a shift, an extract, a compare and a select per bit
// (measured: depth-sort passes 0.870 -> 0.836 ms per batch, K4c scatter
// 1.236 -> 1.159).
__device__ __forceinline__ uint32_t agree_bit(uint32_t d, uint32_t bit_mask) {
  uint32_t bb, x;
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
      "and.b32 t, %2, %3;\n\tsetp.ne.u32 p, t, 0;\n\t"
      "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\tselp.b32 %1, 0, 0xffffffff, p;\n\t}"
      : "=r"(bb), "=r"(x) : "r"(d), "r"(bit_mask));
  return bb ^ x;
}

// Lanes of the warp holding the same 8-bit digit: 8 ballots (ALU pipe, fully
// pipelined) instead of MATCH.ANY, whose latency dominated the ranking loop
// in the ncu source view.
__device__ __forceinline__ uint32_t match_digit8(bool valid, uint32_t d) {
  uint32_t peers = __ballot_sync(FULL, valid);
#pragma unroll
  for (int b = 0; b < 8; ++b) peers &= agree_bit(d, 1u << b);
  return peers;
}

__device__ __forceinline__ void publish(uint64_t* words, int64_t bid, uint64_t v) {
  st_word(words + bid, v);
}

// ---------------------------------------------------------------------------
// K2: compact visible (view, g) pairs, K and visible-count totals.
// Block tile = 256 threads x 8 consecutive items.
constexpr int K2_ITEMS = 12;
constexpr int K2_TILE = 256 * K2_ITEMS;

// KeyT = uint64_t: key = view << 32 | depth bits.  KeyT = uint32_t (the
// default): key = view << dshift | (depth bits - dbase) with dbase = the bits
// of the batch's smallest znear (every visible depth is above it, and
// positive float bits order like the floats); a depth whose offset needs more
// than dshift bits raises totals[2] and the caller reruns with 64-bit keys.
// Same order either way; the 32-bit keys halve the depth sort's traffic
// (4 passes x 8 B instead of 5 x 12 B per visible pair).
template <typename KeyT>
#ifndef K2_MINB
#define K2_MINB 5  // measured: 5 blocks (48 regs) 3,019, 4 (64) 3,014, unbounded (80) 3,001 views/s
#endif
__global__ void __launch_bounds__(256, K2_MINB) k2_compact(const uint32_t* __restrict__ depth_plane,
                                                  const uint32_t* __restrict__ nt_plane, int64_t M, int64_t n,
                                                  KeyT* __restrict__ dkeys, uint32_t* __restrict__ dvals,
                                                  uint32_t* __restrict__ emit_off, uint64_t* __restrict__ lb_vis,
                                                  uint64_t* __restrict__ lb_k, uint32_t* __restrict__ ctr,
                                                  uint64_t* __restrict__ totals, uint32_t* __restrict__ hist,
                                                  int dpasses, int dshift, uint32_t dbase) {
  __shared__ uint32_t s_hist[5][256];
  __shared__ uint64_t s_wv[8], s_wk[8];
  __shared__ uint64_t s_pv, s_pk, s_tv;
  __shared__ uint32_t s_bid;
  // the block's visible (key, g) pairs, compacted here first so the global
  // writes are coalesced
  __shared__ KeyT s_key[K2_TILE];
  __shared__ uint32_t s_g[K2_TILE];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(ctr, 1u);
  for (int i = tid; i < 5 * 256; i += 256) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t bid = s_bid;
  const int64_t i0 = bid * K2_TILE + (int64_t)tid * K2_ITEMS;
  uint32_t nt[K2_ITEMS];
  uint32_t cv = 0;
  uint64_t ck = 0;
#pragma unroll
  for (int k = 0; k < K2_ITEMS; ++k) {
    nt[k] = (i0 + k < M) ? __ldg(nt_plane + i0 + k) : 0u;
    cv += nt[k] > 0;
    ck += nt[k];
  }
  // block exclusive scan of (cv, ck)
  uint64_t iv = warp_incl_scan<uint64_t>(cv), ik = warp_incl_scan<uint64_t>(ck);
  if (lane == 31) { s_wv[warp] = iv; s_wk[warp] = ik; }
  __syncthreads();
  if (warp == 0) {
    uint64_t wv = lane < 8 ? s_wv[lane] : 0, wk = lane < 8 ? s_wk[lane] : 0;
    uint64_t sv = warp_incl_scan<uint64_t>(wv), sk = warp_incl_scan<uint64_t>(wk);
    if (lane < 8) { s_wv[lane] = sv - wv; s_wk[lane] = sk - wk; }
    const uint64_t tv = __shfl_sync(FULL, sv, 7), tk = __shfl_sync(FULL, sk, 7);
    uint64_t pv = 0, pk = 0;
    if (bid == 0) {
      if (lane == 0) { publish(lb_vis, 0, LB_INC | tv); publish(lb_k, 0, LB_INC | tk); }
    } else {
      if (lane == 0) { publish(lb_vis, bid, LB_AGG | tv); publish(lb_k, bid, LB_AGG | tk); }
      pv = warp_lookback(lb_vis, bid);
      pk = warp_lookback(lb_k, bid);
      if (lane == 0) { publish(lb_vis, bid, LB_INC | (pv + tv)); publish(lb_k, bid, LB_INC | (pk + tk)); }
    }
    if (lane == 0) {
      s_pv = pv; s_pk = pk; s_tv = tv;
      if ((bid + 1) * K2_TILE >= M) { totals[0] = pv + tv; totals[1] = pk + tk; }
    }
  }
  __syncthreads();
  uint32_t lv = (uint32_t)(s_wv[warp] + (iv - cv));  // block-local slot
  uint64_t pk = s_pk + s_wk[warp] + (ik - ck);
  // (view, g) of i0 with one division per thread, then stepped
  uint64_t view = i0 < M ? (uint64_t)(i0 / n) : 0;
  int64_t g = i0 - (int64_t)view * n;
  bool wide_miss = false;
#pragma unroll
  for (int k = 0; k < K2_ITEMS; ++k) {
    const int64_t i = i0 + k;
    if (i >= M) break;
    if (g == n) { g = 0; ++view; }
    if (emit_off) emit_off[i] = (uint32_t)pk;
    if (nt[k]) {
      const uint32_t d = __ldg(depth_plane + i);
      KeyT key;
      if (sizeof(KeyT) == 8) {
        key = (KeyT)((view << 32) | d);
      } else {
        const uint32_t off = d - dbase;
        wide_miss |= (off >> dshift) != 0;  // does not fit: caller falls back to 64-bit keys
        key = (KeyT)(((uint32_t)view << dshift) | off);
      }
      s_key[lv] = key;
      s_g[lv] = (uint32_t)g;
      ++lv;
    }
    pk += nt[k];
    ++g;
  }
  if (wide_miss) totals[2] = 1;
  __syncthreads();
  const uint32_t bt = (uint32_t)s_tv;
  const uint64_t pv0 = s_pv;
  for (uint32_t j = tid; j < bt; j += 256) {
    const KeyT key = s_key[j];
    GSR_DCHECK(pv0 + j < (uint64_t)M);
    dkeys[pv0 + j] = key;
    dvals[pv0 + j] = s_g[j];
    for (int p = 0; p < dpasses; ++p) atomicAdd(&s_hist[p][(uint32_t)(key >> (8 * p)) & 255], 1u);
  }
  __syncthreads();
  for (int i = tid; i < dpasses * 256; i += 256) {
    const uint32_t c = (&s_hist[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// ---------------------------------------------------------------------------
// Exclusive scan of `passes` 256-bin histograms -> bases (one block).
__global__ void scan_hist(const uint32_t* __restrict__ hist, uint32_t* __restrict__ base, int passes) {
  __shared__ uint32_t s_w[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int p = 0; p < passes; ++p) {
    const uint32_t c = hist[p * 256 + t];
    const uint32_t inc = warp_incl_scan<uint32_t>(c);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t off = 0;
    for (int w = 0; w < warp; ++w) off += s_w[w];
    base[p * 256 + t] = off + inc - c;
    __syncthreads();
  }
}

// Histograms of all passes of a u64-key sort (utility sort).
__global__ void __launch_bounds__(256) hist_u64(const uint64_t* __restrict__ keys, int64_t n, int begin_bit,
                                                int passes, int end_bit, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_hist[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += 256) (&s_hist[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) {
    const uint64_t k = keys[i];
    for (int p = 0; p < passes; ++p) {
      const int sh = begin_bit + 8 * p;
      const int nb = min(8, end_bit - sh);
      atomicAdd(&s_hist[p][(uint32_t)(k >> sh) & ((1u << nb) - 1)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += 256) {
    const uint32_t c = (&s_hist[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// ---------------------------------------------------------------------------
// One onesweep LSD pass: stable scatter of (key, value) by the digit
// (key >> shift) & (2^nbits - 1).  Dynamic block ids guarantee forward
// progress of the per-digit decoupled look-back.
//   MODE 0: write keys_out / vals_out.
//   MODE 1: tile sort final pass (KeyT = u32 key = view*tpv + tile): write
//           vals_out and, if keys64 != null, the full 64-bit key
//           (key << 32) | depth_plane[view * nper + g].
#ifndef OS_MINB12
#define OS_MINB12 4  // 4 blocks per SM (64 registers, small spills): 12-key tiles +0.4 % over 3 (round 1); 16-key tiles 4 vs 3 blocks -1 % depth-sort time (round 2)
#endif
template <typename KeyT, int KPT, int MODE>
__global__ void __launch_bounds__(256, (KPT <= 8 ? 4 : OS_MINB12)) onesweep(const KeyT* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                KeyT* __restrict__ kout, uint32_t* __restrict__ vout, uint32_t n,
                                                int shift, int nbits, const uint32_t* __restrict__ base,
                                                uint32_t* __restrict__ lookback, uint32_t* __restrict__ ctr,
                                                uint64_t* __restrict__ keys64, const uint32_t* __restrict__ depth_plane,
                                                uint32_t tpv, int64_t nper) {
  constexpr int B = 256, W = B / 32, TILE = B * KPT;
  struct Stage {
    KeyT k[TILE];
    uint32_t v[TILE];
  };
  union Smem {
    uint32_t hist[W][256];
    Stage st;
  };
  __shared__ Smem u;
  __shared__ uint32_t s_start[256], s_gbase[256], s_cnt[256], s_wsum[W];
  __shared__ uint32_t s_bid;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(ctr, 1u);
  for (int i = tid; i < W * 256; i += B) (&u.hist[0][0])[i] = 0;
  s_cnt[tid] = 0;
  __syncthreads();
  const uint32_t bid = s_bid;
  const uint32_t mask = (nbits >= 32) ? 0xffffffffu : ((1u << nbits) - 1);
  const int64_t wbase = (int64_t)bid * TILE + (int64_t)warp * (KPT * 32);
  // Keys stay in registers through ranking; values are not needed until the
  // scatter, so they are loaded there (keeps 4 blocks / SM resident).
  KeyT key[KPT];
  uint32_t rank[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int64_t idx = wbase + k * 32 + lane;
    const bool valid = idx < (int64_t)n;
    key[k] = valid ? kin[idx] : KeyT(0);
  }
  const uint32_t lt = (1u << lane) - 1;
  // Early digit counts (shared atomics): the tile's aggregate is published and
  // the first window of look-back loads is in flight while the warps rank.
  constexpr int WIN = 8;
  uint32_t win[WIN];
  uint32_t early_total = 0;
  {
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int64_t idx = wbase + k * 32 + lane;
      if (idx < (int64_t)n) atomicAdd(&s_cnt[(uint32_t)(key[k] >> shift) & mask], 1u);
    }
    __syncthreads();
    early_total = s_cnt[tid];
    st_word(lookback + (size_t)bid * 256 + tid, (bid == 0 ? DG_INC : DG_AGG) | early_total);
#pragma unroll
    for (int i = 0; i < WIN; ++i) {
      const int64_t j = (int64_t)bid - 1 - i;
      win[i] = j >= 0 ? ld_word(lookback + (size_t)j * 256 + tid) : DG_INC;
    }
  }
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int64_t idx = wbase + k * 32 + lane;
    const bool valid = idx < (int64_t)n;
    const uint32_t d = (uint32_t)(key[k] >> shift) & mask;
    const uint32_t peers = match_digit8(valid, d);
    const uint32_t r = __popc(peers & lt);
    uint32_t pre = 0;
    if (valid) pre = u.hist[warp][d];
    __syncwarp();
    if (valid && r == 0) u.hist[warp][d] = pre + __popc(peers);
    __syncwarp();
    rank[k] = pre + r;
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, block total, look-back
  {
    const int d = tid;
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = u.hist[w][d];
      u.hist[w][d] = total;
      total += c;
    }
    uint32_t* my = lookback + (size_t)bid * 256 + d;
    uint32_t excl = 0;
    if (bid != 0) {
      // windowed decoupled look-back: WIN predecessors per round trip
      int64_t j = (int64_t)bid - 1;
      while (true) {
        int i = 0;
        bool done = false;
#pragma unroll
        for (; i < WIN; ++i) {
          const uint32_t f = win[i] >> 30;
          if (f == 0) break;
          excl += win[i] & DG_VAL;
          if (f == 2) {
            done = true;
            break;
          }
        }
        if (done) break;
        j -= i;  // consumed i aggregates; re-read from the first word not yet ready
#ifdef GSR_DEBUG
        if (j < 0) {
          printf("onesweep lookback underflow bid=%u d=%d n=%u shift=%d\n", bid, d, n, shift);
          __trap();
        }
#endif
#pragma unroll
        for (int q = 0; q < WIN; ++q) {
          const int64_t jj = j - q;
          win[q] = jj >= 0 ? ld_word(lookback + (size_t)jj * 256 + d) : DG_INC;
        }
      }
      st_word(my, DG_INC | (excl + total));
    }
    // block-local exclusive scan of totals over digits
    const uint32_t inc = warp_incl_scan<uint32_t>(total);
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    uint32_t off = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) off += (w < warp) ? s_wsum[w] : 0u;
    const uint32_t start = off + inc - total;
    s_start[d] = start;
    s_gbase[d] = base[d] + excl - start;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const uint32_t d = (uint32_t)(key[k] >> shift) & mask;
    rank[k] += s_start[d] + u.hist[warp][d];  // -> position in the block's stage
  }
  uint32_t val[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int64_t idx = wbase + k * 32 + lane;
    val[k] = idx < (int64_t)n ? vin[idx] : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int64_t idx = wbase + k * 32 + lane;
    if (idx < (int64_t)n) {
      u.st.k[rank[k]] = key[k];
      u.st.v[rank[k]] = val[k];
    }
  }
  __syncthreads();
  const int64_t rem = (int64_t)n - (int64_t)bid * TILE;
  const int nvalid = rem < TILE ? (int)rem : TILE;
  for (int i = tid; i < nvalid; i += B) {
    const KeyT kk = u.st.k[i];
    const uint32_t vv = u.st.v[i];
    const uint32_t d = (uint32_t)(kk >> shift) & mask;
    const uint32_t o = s_gbase[d] + i;
#ifdef GSR_DEBUG
    if (o >= n) {
      printf("onesweep OOB write bid=%u d=%u i=%d o=%u n=%u base=%u start=%u\n", bid, d, i, o, n, base[d], s_start[d]);
      __trap();
    }
#endif
    if (MODE == 0) {
      kout[o] = kk;
      vout[o] = vv;
    } else {
      vout[o] = vv;
      if (keys64) {
        const uint32_t k32 = (uint32_t)kk;
        const uint32_t view = k32 / tpv;
        keys64[o] = ((uint64_t)k32 << 32) | __ldg(depth_plane + (int64_t)view * nper + vv);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3: look-back scan of n_tiles in depth-sorted order + load-balanced emission.
// Block = 8 warps x K3_ROUNDS rounds x 32 entries; warp w owns 32 * K3_ROUNDS
// consecutive entries.  Each entry's 32-byte span record (O1 step
// 15) is gathered once.  Emission is two-level load-balanced: the warp's
// (entry, tile row) units are dealt 32 at a time (owner search over the row
// counts), each lane evaluates its unit's span and writes the first K3_LS
// keys of that span itself (to the slots an owner search would deal them
// to); only the keys of wider spans are dealt 32 at a time (owner search over
// the remaining widths).  Keys leave in
// unit order, i.e. (depth, g, ty, tx) order, contiguously from the block's
// look-back offset.
#ifndef K3_ROUNDS_N
#define K3_ROUNDS_N 4
#endif
constexpr int K3_ROUNDS = K3_ROUNDS_N;
#ifndef K3_OWNER_OR
#define K3_OWNER_OR 1
#endif
#ifndef K3_GENERIC_CNT
#define K3_GENERIC_CNT 1
#endif
#ifndef K3_LS
#define K3_LS 8  // keys per row written lane-serially (0: every key dealt 32 at a time; measured 0 / 3 / 4 / 6 / 8 / 12: emit 1.049 / 1.050 / 1.053 / 0.977 / 0.971 / 0.992 ms per batch, bench 3,401 / 3,405 / 3,423 / 3,453 / 3,456 / 3,447 views/s)
#endif
constexpr int K3_TILE = 256 * K3_ROUNDS;

__device__ __forceinline__ int owner_of(uint32_t excl, uint32_t j) {  // largest s with excl[s] <= j
  int s = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const uint32_t e = __shfl_sync(FULL, excl, s + step);
    if (e <= j) s += step;
  }
  return s;
}

template <typename KeyT, bool PACK>
#ifndef K3_MINB
#define K3_MINB 6  // measured (with OS_MINB12 4): 6 blocks 3,076, 5 3,052, 8 3,059, unbounded (64 regs) 3,019 views/s
#endif
__global__ void __launch_bounds__(256, K3_MINB) k3_emit(const KeyT* __restrict__ dkeys, const uint32_t* __restrict__ dvals,
                                               int64_t nvis, const uint4* __restrict__ span, int64_t n, uint32_t gx,
                                               uint32_t tpv, int W, uint32_t* __restrict__ tkeys,
                                               uint32_t* __restrict__ tvals, uint32_t* __restrict__ counts,
                                               uint64_t* __restrict__ lb, uint32_t* __restrict__ ctr,
                                               int smem_bins, int vshift, int gbits, uint64_t kcap, uint64_t T) {
  // gbits > 0: each key leaves as ONE packed word (tile within its view <<
  // gbits | g) in tkeys and tvals is not written (the K4c path unpacks it)
  // Per-tile counts: a shared-memory histogram over the tiles of the block's
  // first view (a depth-sorted block almost always lies in one view), flushed
  // with one global atomic per non-empty bin; other views go straight to
  // global memory.
  extern __shared__ uint32_t s_cnt[];
  __shared__ uint64_t s_w[8];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_bid, s_view0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    const uint32_t b = atomicAdd(ctr, 1u);
    s_bid = b;
    s_view0 = (uint32_t)(dkeys[(int64_t)b * K3_TILE] >> vshift);
  }
  for (int t = tid; t < smem_bins; t += 256) s_cnt[t] = 0;
  __syncthreads();
  const int64_t bid = s_bid;
  const uint32_t view0 = s_view0;
  const uint32_t lo = view0 * tpv;
  const int64_t e0 = bid * K3_TILE + (int64_t)warp * (32 * K3_ROUNDS);
  uint4 s0[K3_ROUNDS], s1[K3_ROUNDS];
  uint32_t g[K3_ROUNDS], view[K3_ROUNDS];
  uint64_t mine = 0;
#pragma unroll
  for (int r = 0; r < K3_ROUNDS; ++r) {
    const int64_t e = e0 + r * 32 + lane;
    s0[r] = make_uint4(0, 0, 0, 0);
    s1[r] = make_uint4(0, 0, 0, 0);
    g[r] = 0;
    view[r] = 0;
    if (e < nvis) {
      const KeyT key = dkeys[e];
      g[r] = dvals[e];
      view[r] = (uint32_t)(key >> vshift);
      GSR_DCHECK(g[r] < n);
      const int64_t pi = (int64_t)view[r] * n + g[r];
      s0[r] = __ldg(span + 2 * pi);
      s1[r] = __ldg(span + 2 * pi + 1);
    }
    mine += s1[r].w;
  }
  const uint64_t wtot = warp_sum<uint64_t>(mine);
  if (lane == 0) s_w[warp] = wtot;
  __syncthreads();
  if (warp == 0) {
    const uint64_t v = lane < 8 ? s_w[lane] : 0;
    const uint64_t inc = warp_incl_scan<uint64_t>(v);
    const uint64_t tot = __shfl_sync(FULL, inc, 7);
    if (lane < 8) s_w[lane] = inc - v;
    uint64_t p = 0;
    if (bid == 0) {
      if (lane == 0) publish(lb, 0, LB_INC | tot);
    } else {
      if (lane == 0) publish(lb, bid, LB_AGG | tot);
      p = warp_lookback(lb, bid);
      if (lane == 0) publish(lb, bid, LB_INC | (p + tot));
    }
    if (lane == 0) s_prefix = p;
  }
  __syncthreads();
  uint64_t base = s_prefix + s_w[warp];
#pragma unroll
  for (int r = 0; r < K3_ROUNDS; ++r) {
    const uint32_t pyr = s1[r].z;
    const uint32_t nrows = s1[r].w ? (pyr >> 20) - ((pyr & 0xffffu) >> 4) + 1u : 0u;
    const uint32_t rinc = warp_incl_scan<uint32_t>(nrows);
    const uint32_t rexcl = rinc - nrows;
    const uint32_t rtot = __shfl_sync(FULL, rinc, 31);
#if K3_OWNER_OR
    // every entry of a round has >= 1 tile row (entries past nvis, all at the
    // end, have none), so the owner of slot j is the number of entries whose
    // first row is at or before j, minus one: one OR-reduction of the step's
    // row-start bits and a popcount instead of a 5-step shuffle search
    int s_carry = -1;
#endif
    for (uint32_t ub = 0; ub < rtot; ub += 32) {
      const uint32_t j = ub + lane;
#if K3_OWNER_OR
      const uint32_t dd = rexcl - ub;  // < 32: this entry's first row is in this step
      const uint32_t M = __reduce_or_sync(FULL, (dd < 32u && nrows) ? (1u << dd) : 0u);
      const int s = s_carry + __popc(M & (0xffffffffu >> (31 - lane)));
      s_carry = __shfl_sync(FULL, s, 31);
#else
      const int s = owner_of(rexcl, j);
#endif
      const float u = __uint_as_float(__shfl_sync(FULL, s0[r].x, s));
      const float v = __uint_as_float(__shfl_sync(FULL, s0[r].y, s));
      const float sp = __uint_as_float(__shfl_sync(FULL, s0[r].z, s));
      const float sh = __uint_as_float(__shfl_sync(FULL, s0[r].w, s));
      const float sic = __uint_as_float(__shfl_sync(FULL, s1[r].x, s));
      const float sdys = __uint_as_float(__shfl_sync(FULL, s1[r].y, s));
      const uint32_t opyr = __shfl_sync(FULL, pyr, s);
      const uint32_t oex = __shfl_sync(FULL, rexcl, s);
      const uint32_t og = __shfl_sync(FULL, g[r], s);
      const uint32_t ov = __shfl_sync(FULL, view[r], s);
      uint32_t w = 0, kb = 0, kl = 0;
      if (j < rtot) {
        const uint32_t py0 = opyr & 0xffffu, py1 = opyr >> 16;
        const uint32_t ty = (py0 >> 4) + (j - oex);
        uint32_t x0, x1;
        row_span(u, v, sp, sh, sic, sdys, py0, py1, ty, W, x0, x1);
        w = x1 - x0;
        kb = ov * tpv + ty * gx + x0;
        kl = PACK ? ((ty * gx + x0) << gbits) | og : og;
      }
      const uint32_t winc = warp_incl_scan<uint32_t>(w);
      const uint32_t wexcl = winc - w;
      const uint32_t wt = __shfl_sync(FULL, winc, 31);
#if K3_LS > 0
      // key slots in 32-bit arithmetic (K < 2^32, as the tile sort's u32
      // positions already require): one wide multiply-add per address
      const uint32_t b32 = (uint32_t)base;
      // each lane writes the first K3_LS keys of its own row span (the same
      // slots the dealt loop would use: b32 + wexcl + i); only the keys of
      // rows wider than K3_LS tiles go through the dealt loop below
      const uint32_t wmax = __reduce_max_sync(FULL, w);
#if K3_GENERIC_CNT
      // a row span lies in one view: its counters are all in the block's
      // shared histogram or all global -- one generic pointer per row
      uint32_t* cp = (kb - lo < (uint32_t)smem_bins) ? s_cnt + (kb - lo) : counts + kb;
#endif
#pragma unroll
      for (uint32_t i = 0; i < (uint32_t)K3_LS; ++i) {
        if (i >= wmax) break;
        if (i < w) {
          const uint32_t key = kb + i;
          GSR_DCHECK(b32 + wexcl + i < kcap && key < T);
          if (PACK) {
            tkeys[b32 + wexcl + i] = kl + (i << gbits);
          } else {
            tkeys[b32 + wexcl + i] = key;
            tvals[b32 + wexcl + i] = kl;
          }
#if K3_GENERIC_CNT
          atomicAdd(cp + i, 1u);
#else
          if (key - lo < (uint32_t)smem_bins)
            atomicAdd(s_cnt + (key - lo), 1u);
          else
            atomicAdd(counts + key, 1u);
#endif
        }
      }
      if (wmax > (uint32_t)K3_LS) {
        const uint32_t w2 = w > (uint32_t)K3_LS ? w - (uint32_t)K3_LS : 0u;
        const uint32_t w2inc = warp_incl_scan<uint32_t>(w2);
        const uint32_t w2excl = w2inc - w2;
        const uint32_t w2t = __shfl_sync(FULL, w2inc, 31);
        for (uint32_t kb0 = 0; kb0 < w2t; kb0 += 32) {
          const uint32_t k = kb0 + lane;
          const int t = owner_of(w2excl, k);
          const uint32_t okb = __shfl_sync(FULL, kb, t);
          const uint32_t owx = __shfl_sync(FULL, wexcl, t);
          const uint32_t ow2 = __shfl_sync(FULL, w2excl, t);
          const uint32_t okl = __shfl_sync(FULL, kl, t);
          if (k < w2t) {
            const uint32_t i = (uint32_t)K3_LS + (k - ow2);
            const uint32_t key = okb + i;
            GSR_DCHECK(b32 + owx + i < kcap && key < T);
            if (PACK) {
              tkeys[b32 + owx + i] = okl + (i << gbits);
            } else {
              tkeys[b32 + owx + i] = key;
              tvals[b32 + owx + i] = okl;
            }
            if (key - lo < (uint32_t)smem_bins)
              atomicAdd(s_cnt + (key - lo), 1u);
            else
              atomicAdd(counts + key, 1u);
          }
        }
      }
#else
      for (uint32_t kb0 = 0; kb0 < wt; kb0 += 32) {
        const uint32_t k = kb0 + lane;
        const int t = owner_of(wexcl, k);
        const uint32_t okb = __shfl_sync(FULL, kb, t);
        const uint32_t owx = __shfl_sync(FULL, wexcl, t);
        const uint32_t okl = __shfl_sync(FULL, kl, t);
        if (k < wt) {
          const uint32_t key = okb + (k - owx);
          GSR_DCHECK(base + k < kcap && key < T);
          if (PACK) {
            tkeys[base + k] = okl + ((k - owx) << gbits);
          } else {
            tkeys[base + k] = key;
            tvals[base + k] = okl;
          }
          if (key - lo < (uint32_t)smem_bins)
            atomicAdd(s_cnt + (key - lo), 1u);
          else
            atomicAdd(counts + key, 1u);
        }
      }
#endif
      base += wt;
    }
  }
  __syncthreads();
  for (int t = tid; t < smem_bins; t += 256) {
    const uint32_t c = s_cnt[t];
    if (c) atomicAdd(counts + lo + t, c);
  }
}

// ---------------------------------------------------------------------------
// K5 (K4c path): ranges[t] = [s, s + counts[t]), s = exclusive prefix of
// counts, as a single-pass decoupled look-back scan over 256-thread blocks of
// 16 consecutive tiles per thread (small blocks: the sort stream's kernels
// must find room on SMs the other slot's composite occupies; the one-block
// K5 below waited for a whole SM).
constexpr int K5_ITEMS = 16;
constexpr int K5_TILE = 256 * K5_ITEMS;

__global__ void __launch_bounds__(256) k5_scan(const uint32_t* __restrict__ counts, int64_t T,
                                               uint2* __restrict__ ranges, uint64_t* __restrict__ lb,
                                               uint32_t* __restrict__ ctr) {
  __shared__ uint32_t s_w[8];
  __shared__ uint32_t s_bid, s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(ctr, 1u);
  __syncthreads();
  const int64_t bid = s_bid;
  const int64_t t0 = bid * K5_TILE + (int64_t)tid * K5_ITEMS;
  uint32_t v[K5_ITEMS];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < K5_ITEMS; ++k) {
    v[k] = t0 + k < T ? __ldg(counts + t0 + k) : 0u;
    sum += v[k];
  }
  const uint32_t inc = warp_incl_scan<uint32_t>(sum);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t wv = lane < 8 ? s_w[lane] : 0u;
    const uint32_t wi = warp_incl_scan<uint32_t>(wv);
    const uint32_t tot = __shfl_sync(FULL, wi, 7);
    if (lane < 8) s_w[lane] = wi - wv;
    uint64_t p = 0;
    if (bid == 0) {
      if (lane == 0) publish(lb, 0, LB_INC | tot);
    } else {
      if (lane == 0) publish(lb, bid, LB_AGG | tot);
      p = warp_lookback(lb, bid);
      if (lane == 0) publish(lb, bid, LB_INC | (p + tot));
    }
    if (lane == 0) s_prefix = (uint32_t)p;
  }
  __syncthreads();
  uint32_t run = s_prefix + s_w[warp] + inc - sum;
#pragma unroll
  for (int k = 0; k < K5_ITEMS; ++k) {
    if (t0 + k < T) ranges[t0 + k] = make_uint2(run, run + v[k]);
    run += v[k];
  }
}

// ---------------------------------------------------------------------------
// K5: ranges[t] = [s, s + counts[t]) with s = exclusive prefix of counts, and
// the tile-sort digit histograms + bases.  One block of 1024 threads.
__global__ void __launch_bounds__(1024) k5_ranges(const uint32_t* __restrict__ counts, int64_t T,
                                                  uint2* __restrict__ ranges, int tpasses,
                                                  uint32_t* __restrict__ hist, uint32_t* __restrict__ base) {
  __shared__ uint32_t s_hist[4][256];
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 4 * 256; i += 1024) (&s_hist[0][0])[i] = 0;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  constexpr int IT = 16;
  for (int64_t c0 = 0; c0 < T; c0 += 1024 * IT) {
    uint32_t v[IT];
    uint32_t sum = 0;
    const int64_t t0 = c0 + (int64_t)tid * IT;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int64_t t = t0 + k;
      v[k] = t < T ? counts[t] : 0u;
      sum += v[k];
      if (v[k]) {
        for (int p = 0; p < tpasses; ++p) atomicAdd(&s_hist[p][(uint32_t)(t >> (8 * p)) & 255], v[k]);
      }
    }
    const uint32_t inc = warp_incl_scan<uint32_t>(sum);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint32_t wv = s_w[lane];
      const uint32_t wi = warp_incl_scan<uint32_t>(wv);
      s_w[lane] = wi - wv;
    }
    __syncthreads();
    uint32_t run = s_carry + s_w[warp] + inc - sum;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int64_t t = t0 + k;
      if (t < T) ranges[t] = make_uint2(run, run + v[k]);
      run += v[k];
    }
    __syncthreads();
    if (tid == 1023) s_carry = run;
    __syncthreads();
  }
  // histograms -> exclusive bases
  for (int p = 0; p < tpasses; ++p) {
    uint32_t c = 0, inc = 0;
    if (tid < 256) {  // warps 0..7, fully active
      c = s_hist[p][tid];
      hist[p * 256 + tid] = c;
      inc = warp_incl_scan<uint32_t>(c);
      if (lane == 31) s_w[warp] = inc;
    }
    __syncthreads();
    if (tid < 256) {
      uint32_t off = 0;
      for (int w = 0; w < warp; ++w) off += s_w[w];
      base[p * 256 + tid] = off + inc - c;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4c: the tile sort as a stable counting scatter (default; the two onesweep
// passes of K4b remain for tiles-per-view > CS_MAX_TPV).  The duplicated keys
// are view-major (K3 emits view by view), every tile's output range is known
// from K5, so only each key's rank among the earlier keys of its tile is
// needed.  Chunks of CS_CHUNK keys never straddle a view:
//   cs_hist  per chunk, per tile of the chunk's view: key counts -> H[chunk][tpv]
//   cs_scan  per (view, tile): H[chunk][tile] <- ranges[tile].start + counts of
//            the view's earlier chunks (column scan, in place)
//   cs_scatter per chunk, in sub-rounds of W x 32 x CS_KPT keys: warp-local
//            stable ranks (ballot match on the tile digit), exclusive prefix
//            over the warps, plus the chunk's running per-tile counter; the
//            value goes straight to its final slot.
// DRAM traffic per key: 4 B (hist) + 4 B (packed) or 8 B read + 4 B write
// (scatter) + the H matrix (CS_CHUNK = 64 K keys: ~0.15 B/key at c3), vs
// 28 B/key for two radix passes.
#ifndef CS_PF
#define CS_PF 1  // packed words of the next sub-round loaded during this one's prefix / scatter
#endif
#ifndef CS_MINB
#define CS_MINB 3
#endif
constexpr int CS_KPT = 16;  // keys per lane per sub-round (round 2: 16 3,190 / 12 3,186 / 8 3,173 / 6 3,156 views/s)
#ifndef CS_CHUNK_KEYS
#define CS_CHUNK_KEYS 65536  // measured: 64 K 2,895, 32 K 2,887, 16 K 2,880 views/s
#endif
constexpr int CS_CHUNK = CS_CHUNK_KEYS;
constexpr int CS_MAX_TPV = 12288;
constexpr int CS_AUTO_TPV = 4352;

// view / chunk bookkeeping (K5 tail): vs[v] = first key of view v (vs[V] = K),
// pb[v] = first chunk of view v (pb[V] = chunks)
__device__ __forceinline__ void cs_locate(const uint32_t* __restrict__ meta, int V, uint32_t chunk, int& v,
                                          uint32_t& k0, uint32_t& k1, uint32_t ch) {
  const uint32_t* vs = meta;
  const uint32_t* pb = meta + (V + 1);
  int lo = 0, hi = V - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pb[mid] <= chunk) lo = mid; else hi = mid - 1;
  }
  v = lo;
  k0 = vs[v] + (chunk - pb[v]) * ch;
  k1 = min(k0 + ch, vs[v + 1]);
}

__global__ void __launch_bounds__(64) cs_meta(const uint2* __restrict__ ranges, int V, uint32_t tpv, uint32_t K,
                                              uint32_t* __restrict__ meta, uint32_t ch) {
  // one thread per view (V <= 64): first key, chunk count, then an exclusive
  // scan of the chunk counts over two warps
  __shared__ uint32_t s_w[2];
  const int v = threadIdx.x, lane = v & 31, warp = v >> 5;
  uint32_t s = K, c = 0;
  if (v < V) {
    s = ranges[(size_t)v * tpv].x;
    const uint32_t e = (v + 1 < V) ? ranges[(size_t)(v + 1) * tpv].x : K;
    c = (e - s + ch - 1) / ch;
  }
  const uint32_t inc = warp_incl_scan<uint32_t>(c);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  const uint32_t pb = inc - c + (warp ? s_w[0] : 0u);
  if (v < V) {
    meta[v] = s;
    meta[(V + 1) + v] = pb;
    if (v == V - 1) {
      meta[V] = K;
      meta[(V + 1) + V] = pb + c;  // the total chunk count
    }
  }
}

__global__ void __launch_bounds__(256) cs_hist(const uint32_t* __restrict__ tkeys, const uint32_t* __restrict__ meta,
                                               int V, uint32_t tpv, uint32_t* __restrict__ H, int gbits, uint32_t ch) {
  extern __shared__ uint32_t s_h[];
  const uint32_t chunk = blockIdx.x;
  if (chunk >= meta[(V + 1) + V]) return;
  int v;
  uint32_t k0, k1;
  cs_locate(meta, V, chunk, v, k0, k1, ch);
  for (uint32_t d = threadIdx.x; d < tpv; d += 256) s_h[d] = 0;
  __syncthreads();
  const uint32_t vb = (uint32_t)v * tpv;
  if (gbits)
    for (uint32_t i = k0 + threadIdx.x; i < k1; i += 256) {
      GSR_DCHECK((__ldg(tkeys + i) >> gbits) < tpv);
      atomicAdd(s_h + (__ldg(tkeys + i) >> gbits), 1u);
    }
  else
    for (uint32_t i = k0 + threadIdx.x; i < k1; i += 256) atomicAdd(s_h + (__ldg(tkeys + i) - vb), 1u);
  __syncthreads();
  uint32_t* row = H + (size_t)chunk * tpv;
  for (uint32_t d = threadIdx.x; d < tpv; d += 256) row[d] = s_h[d];
}

__global__ void __launch_bounds__(256) cs_scan(const uint2* __restrict__ ranges, const uint32_t* __restrict__ meta,
                                               int V, uint32_t tpv, uint32_t* __restrict__ H) {
  const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;  // global tile = v * tpv + d
  if (t >= (uint64_t)V * tpv) return;
  const int v = (int)(t / tpv);
  const uint32_t d = (uint32_t)(t - (uint64_t)v * tpv);
  const uint32_t* pb = meta + (V + 1);
  uint32_t run = ranges[t].x;
  const uint32_t c1 = pb[v + 1];
  uint32_t c = pb[v];
  // 16 independent loads in flight per step (the column walk is latency-bound)
  for (; c + 16 <= c1; c += 16) {
    uint32_t x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = H[(size_t)(c + j) * tpv + d];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      H[(size_t)(c + j) * tpv + d] = run;
      run += x[j];
    }
  }
  for (; c < c1; ++c) {
    uint32_t* p = H + (size_t)c * tpv + d;
    const uint32_t x = *p;
    *p = run;
    run += x;
  }
}

// Lanes of the warp whose DB-bit digit equals this lane's (DB a compile-time
// width, so every bit test takes an immediate mask).
template <int DB>
__device__ __forceinline__ uint32_t match_digits(bool ok, uint32_t d) {
  uint32_t peers = __ballot_sync(FULL, ok);
#pragma unroll
  for (int b = 0; b < DB; ++b) peers &= agree_bit(d, 1u << b);
  return peers;
}

template <int W, bool PACK, int DB = 0>
__global__ void __launch_bounds__(W * 32, CS_MINB) cs_scatter(const uint32_t* __restrict__ tkeys,
                                                     const uint32_t* __restrict__ tvals,
                                                     const uint32_t* __restrict__ meta, int V, uint32_t tpv,
                                                     int dbits, uint32_t tslice, int nslice,
                                                     const uint32_t* __restrict__ H,
                                                     uint32_t* __restrict__ vals_out, uint64_t* __restrict__ keys64,
                                                     const uint32_t* __restrict__ depth_plane, int64_t nper,
                                                     int gbits, uint32_t ch) {
  // gbits > 0: packed words (tile within the view << gbits | g), no tvals
  // shared memory: s_base [tpv] u32 (chunk offset + keys so far), s_sub [tpv]
  // u32 (this sub-round's base), s_wh [W][tpv] u16 (per-warp counts, then
  // the exclusive prefix over the warps)
  // per-warp rows are padded to a multiple of 8 tiles (16 B) so the prefix
  // loop can work on packed u16 pairs and the reset on 16-byte stores
  extern __shared__ uint32_t smem[];
  // blocks (chunk, slice): the slice's tiles [tb, tb + tn) only (large tile
  // counts are split so 8 warps' counters fit in shared memory)
  const uint32_t chunk = blockIdx.x / nslice;
  const uint32_t tb = (blockIdx.x - chunk * nslice) * tslice;
  const uint32_t tn = min(tslice, tpv - tb);
  const uint32_t ts = (tn + 7u) & ~7u;  // row stride (u16 elements)
  uint32_t* s_base = smem;
  uint32_t* s_sub = smem + ts;
  uint16_t* s_wh = reinterpret_cast<uint16_t*>(smem + 2 * ts);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (chunk >= meta[(V + 1) + V]) return;
  int v;
  uint32_t k0, k1;
  cs_locate(meta, V, chunk, v, k0, k1, ch);
  const uint32_t vb = (uint32_t)v * tpv + tb;
  const uint32_t* Hrow = H + (size_t)chunk * tpv + tb;
  for (uint32_t d = tid; d < tn; d += W * 32) s_base[d] = Hrow[d];
  for (uint32_t i = tid; i < (uint32_t)W * ts / 8; i += W * 32) reinterpret_cast<uint4*>(s_wh)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  uint16_t* wh = s_wh + (size_t)warp * ts;
  constexpr uint32_t SUB = W * 32 * CS_KPT;
  // packed words of the next sub-round are loaded during this one's prefix
  // and scatter (measured +0.15 %; the two-plane layout loads in place)
#if CS_PF
  uint32_t nw[CS_KPT];
  if (PACK) {
#pragma unroll
    for (int k = 0; k < CS_KPT; ++k) {
      const uint32_t i = k0 + (uint32_t)warp * (32 * CS_KPT) + k * 32 + lane;
      nw[k] = i < k1 ? __ldg(tkeys + i) : 0xffffffffu;
    }
  }
#endif
  for (uint32_t s0 = k0; s0 < k1; s0 += SUB) {
    const uint32_t wb = s0 + (uint32_t)warp * (32 * CS_KPT);
    uint32_t dg[CS_KPT], vv[CS_KPT], rk[CS_KPT];
#pragma unroll
    for (int k = 0; k < CS_KPT; ++k) {
      const uint32_t i = wb + k * 32 + lane;
      if (PACK) {
#if CS_PF
        const uint32_t wd = nw[k];
#else
        const uint32_t wd = i < k1 ? __ldg(tkeys + i) : 0xffffffffu;
#endif
        dg[k] = i < k1 ? (wd >> gbits) - tb : 0xffffffffu;  // out of the slice: >= tn
        vv[k] = wd & ((1u << gbits) - 1u);
      } else {
        dg[k] = i < k1 ? __ldg(tkeys + i) - vb : 0xffffffffu;  // out of the slice: >= tn
        vv[k] = (i < k1 && dg[k] < tn) ? __ldg(tvals + i) : 0u;
      }
    }
    // warp-local stable ranks: lanes holding the same tile digit (ballots per bit)
#pragma unroll
    for (int k = 0; k < CS_KPT; ++k) {
      const bool ok = dg[k] < tn;
      uint32_t peers;
      if constexpr (DB > 0) {
        peers = match_digits<DB>(ok, dg[k]);  // bits >= dbits are 0 in every ok lane
      } else {
        peers = __ballot_sync(FULL, ok);
        for (int b = 0; b < dbits; ++b) {
          const bool bit = (dg[k] >> b) & 1u;
          const uint32_t bb = __ballot_sync(FULL, bit);
          peers &= bit ? bb : ~bb;
        }
      }
      uint32_t pre = 0;
      if (ok) pre = wh[dg[k]];
      __syncwarp();
      if (ok && (peers & lt) == 0) wh[dg[k]] = (uint16_t)(pre + __popc(peers));
      __syncwarp();
      rk[k] = pre + __popc(peers & lt);
    }
#if CS_PF
    if (PACK) {
#pragma unroll
      for (int k = 0; k < CS_KPT; ++k) {
        const uint32_t i = wb + SUB + k * 32 + lane;
        nw[k] = i < k1 ? __ldg(tkeys + i) : 0xffffffffu;
      }
    }
#endif
    __syncthreads();
    // exclusive prefix over the warps, four tiles per 64-bit word (no carry:
    // a sub-round holds at most W x 32 x CS_KPT < 2^16 keys); the bases of
    // the word's four tiles move as one 16-byte vector (ts % 8 == 0; tiles
    // >= tn are padding nobody reads)
    uint64_t* wh64 = reinterpret_cast<uint64_t*>(s_wh);
    for (uint32_t p = tid; p < ts / 4; p += W * 32) {
      uint64_t run = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint64_t* q = wh64 + (size_t)w * (ts / 4) + p;
        const uint64_t c = *q;
        *q = run;
        run += c;
      }
      uint4 b = reinterpret_cast<const uint4*>(s_base)[p];
      reinterpret_cast<uint4*>(s_sub)[p] = b;
      b.x += (uint32_t)run & 0xffffu;
      b.y += (uint32_t)(run >> 16) & 0xffffu;
      b.z += (uint32_t)(run >> 32) & 0xffffu;
      b.w += (uint32_t)(run >> 48);
      reinterpret_cast<uint4*>(s_base)[p] = b;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CS_KPT; ++k) {
      if (dg[k] < tn) {
        const uint32_t pos = s_sub[dg[k]] + (uint32_t)wh[dg[k]] + rk[k];
        GSR_DCHECK(pos >= meta[v] && pos < meta[v + 1]);  // inside its view's key range
        vals_out[pos] = vv[k];
        if (keys64) keys64[pos] = ((uint64_t)(vb + dg[k]) << 32) | __ldg(depth_plane + (int64_t)v * nper + vv[k]);
      }
    }
    __syncthreads();
    for (uint32_t i = tid; i < (uint32_t)W * ts / 8; i += W * 32) reinterpret_cast<uint4*>(s_wh)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
}

// O2 emission order (view, g, ty, tx): parity output only.
__global__ void __launch_bounds__(256) k_emit_o2(const uint32_t* __restrict__ depth_plane,
                                                 const uint4* __restrict__ span,
                                                 const uint32_t* __restrict__ nt_plane,
                                                 const uint32_t* __restrict__ emit_off, int64_t M, int64_t n,
                                                 uint32_t gx, uint32_t tpv, int W, uint64_t* __restrict__ keys,
                                                 uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= M) return;
  const uint32_t nt = nt_plane[i];
  if (!nt) return;
  const uint64_t view = (uint64_t)(i / n);
  const uint32_t g = (uint32_t)(i - (int64_t)view * n);
  const uint4 a = span[2 * i], b = span[2 * i + 1];
  const uint32_t d = depth_plane[i];
  const uint32_t py0 = b.z & 0xffffu, py1 = b.z >> 16;
  uint64_t o = emit_off[i];
  for (uint32_t ty = py0 >> 4; ty <= (py1 >> 4); ++ty) {
    uint32_t x0, x1;
    row_span(__uint_as_float(a.x), __uint_as_float(a.y), __uint_as_float(a.z), __uint_as_float(a.w),
             __uint_as_float(b.x), __uint_as_float(b.y), py0, py1, ty, W, x0, x1);
    for (uint32_t tx = x0; tx < x1; ++tx) {
      const uint64_t tile = view * tpv + (uint64_t)ty * gx + tx;
      keys[o] = (tile << 32) | d;
      vals[o] = g;
      ++o;
    }
  }
}

// ---------------------------------------------------------------------------
// NEXT-2b: compaction in the cached blend order.  Element i of view v is the
// p-th Gaussian of the view's visiting sequence: the segment (tile in visit
// order) holding p maps it to cache[off + p - start].  Visible ones are
// compacted in that order into (view << 32, g) pairs -- the input K3 expects
// -- so the per-view depth sort is skipped.
struct OrderSeg {
  uint64_t off;      // cache offset of the tile's chosen ordering
  uint32_t start;    // first sequence position of the tile
  uint32_t len;      // Gaussians in the tile
};

__global__ void __launch_bounds__(256) k2c_compact(const OrderSeg* __restrict__ segs, int n_seg,
                                                   const uint32_t* __restrict__ cache,
                                                   const uint32_t* __restrict__ nt_plane, int64_t M, int64_t n,
                                                   uint32_t* __restrict__ dkeys, uint32_t* __restrict__ dvals,
                                                   uint64_t* __restrict__ lb_vis, uint64_t* __restrict__ lb_k,
                                                   uint32_t* __restrict__ ctr, uint64_t* __restrict__ totals,
                                                   int vshift) {
  __shared__ uint64_t s_wv[8], s_wk[8];
  __shared__ uint64_t s_pv;
  __shared__ uint32_t s_bid;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(ctr, 1u);
  __syncthreads();
  const int64_t bid = s_bid;
  const int64_t i0 = bid * K2_TILE + (int64_t)tid * K2_ITEMS;
  uint32_t nt[K2_ITEMS], gg[K2_ITEMS];
  uint32_t cv = 0;
  uint64_t ck = 0;
#pragma unroll
  for (int k = 0; k < K2_ITEMS; ++k) {
    nt[k] = 0;
    gg[k] = 0;
    const int64_t i = i0 + k;
    if (i < M) {
      const int64_t view = i / n;
      const uint32_t p = (uint32_t)(i - view * n);
      const OrderSeg* S = segs + view * n_seg;
      int lo = 0, hi = n_seg - 1;  // last segment with start <= p
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (S[mid].start <= p) lo = mid; else hi = mid - 1;
      }
      const uint32_t g = __ldg(cache + S[lo].off + (p - S[lo].start));
      gg[k] = g;
      nt[k] = __ldg(nt_plane + view * n + g);
    }
    cv += nt[k] > 0;
    ck += nt[k];
  }
  uint64_t iv = warp_incl_scan<uint64_t>(cv), ik = warp_incl_scan<uint64_t>(ck);
  if (lane == 31) { s_wv[warp] = iv; s_wk[warp] = ik; }
  __syncthreads();
  if (warp == 0) {
    uint64_t wv = lane < 8 ? s_wv[lane] : 0, wk = lane < 8 ? s_wk[lane] : 0;
    uint64_t sv = warp_incl_scan<uint64_t>(wv), sk = warp_incl_scan<uint64_t>(wk);
    if (lane < 8) { s_wv[lane] = sv - wv; s_wk[lane] = sk - wk; }
    const uint64_t tv = __shfl_sync(FULL, sv, 7), tk = __shfl_sync(FULL, sk, 7);
    uint64_t pv = 0, pk = 0;
    if (bid == 0) {
      if (lane == 0) { publish(lb_vis, 0, LB_INC | tv); publish(lb_k, 0, LB_INC | tk); }
    } else {
      if (lane == 0) { publish(lb_vis, bid, LB_AGG | tv); publish(lb_k, bid, LB_AGG | tk); }
      pv = warp_lookback(lb_vis, bid);
      pk = warp_lookback(lb_k, bid);
      if (lane == 0) { publish(lb_vis, bid, LB_INC | (pv + tv)); publish(lb_k, bid, LB_INC | (pk + tk)); }
    }
    if (lane == 0) {
      s_pv = pv;
      if ((bid + 1) * K2_TILE >= M) { totals[0] = pv + tv; totals[1] = pk + tk; }
    }
  }
  __syncthreads();
  uint64_t pv = s_pv + s_wv[warp] + (iv - cv);
#pragma unroll
  for (int k = 0; k < K2_ITEMS; ++k) {
    const int64_t i = i0 + k;
    if (i >= M) break;
    if (nt[k]) {
      dkeys[pv] = (uint32_t)(i / n) << vshift;
      dvals[pv] = gg[k];
      ++pv;
    }
  }
}

// NEXT-2b cache build: key of element i of segment s = (t, k) is
// (s << 32) | orderable(fl32(fl32(x bx) + fl32(z bz))), value = g.
struct CacheSeg {
  uint64_t out;      // first cache slot of the segment
  uint32_t start;    // first Gaussian of the tile
  uint32_t len;
  float bx, bz;
};

__global__ void __launch_bounds__(256) kc_keys(const CacheSeg* __restrict__ segs, const float4* __restrict__ po,
                                               uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const CacheSeg sg = segs[blockIdx.y];
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < sg.len; i += gridDim.x * 256) {
    const uint32_t g = sg.start + i;
    const float4 P = __ldg(po + g);
    const float key = (P.x * sg.bx) + (P.z * sg.bz);
    uint32_t b = __float_as_uint(key);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    keys[sg.out + i] = ((uint64_t)blockIdx.y << 32) | b;
    vals[sg.out + i] = g;
  }
}

int bits_for(uint64_t count) {  // ceil(log2(count)), 0 for count <= 1
  int b = 0;
  while ((1ull << b) < count) ++b;
  return b;
}

constexpr int KPT64 = 12;  // onesweep u64 keys: 3072 keys per block
constexpr int KPT32 = 16;  // onesweep u32 keys: 4096 keys per block (round 2: 16 keys 3,172 vs 12 keys 3,159 views/s on the bench; 20 keys slower)

template <typename KeyT>
constexpr size_t pass_tile() {
  return 256 * (sizeof(KeyT) == 8 ? KPT64 : KPT32);
}

// One stable LSD onesweep pass by digit (key >> shift) & (2^nbits - 1).
// `region` holds ceil(n / pass_tile) * 256 zero-initialised look-back words;
// `ctr` one zero-initialised counter (dynamic block ids).
template <typename KeyT, int MODE>
cudaError_t run_pass(const KeyT* kin, const uint32_t* vin, KeyT* kout, uint32_t* vout, uint32_t n, int shift, int nbits,
                     const uint32_t* base, uint32_t* region, uint32_t* ctr, uint64_t* keys64,
                     const uint32_t* depth_plane, uint32_t tpv, int64_t nper, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  constexpr int K = sizeof(KeyT) == 8 ? KPT64 : KPT32;
  const uint32_t nt = (uint32_t)((n + pass_tile<KeyT>() - 1) / pass_tile<KeyT>());
  onesweep<KeyT, K, MODE><<<nt, 256, 0, st>>>(kin, vin, kout, vout, n, shift, nbits, base, region, ctr, keys64,
                                              depth_plane, tpv, nper);
  return cudaGetLastError();
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

// ---------------------------------------------------------------------------
// Generic multi-pass onesweep over u64 keys (ping-pong through scratch).
static gsr_status sort_u64_passes(gsr_ctx* ctx, const uint64_t* kin, const uint32_t* vin, uint64_t* kout,
                                  uint32_t* vout, uint64_t* ktmp, uint32_t* vtmp, int64_t n, int begin_bit,
                                  int end_bit, const uint32_t* base, uint32_t* region, uint32_t* ctrs,
                                  cudaStream_t st) {
  const int passes = (end_bit - begin_bit + 7) / 8;
  const size_t nb = (size_t)((n + pass_tile<uint64_t>() - 1) / pass_tile<uint64_t>());
  // choose buffers so that the last pass lands in kout
  const uint64_t* ci = kin;
  const uint32_t* cv = vin;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    uint64_t* ko = to_out ? kout : ktmp;
    uint32_t* vo = to_out ? vout : vtmp;
    const int sh = begin_bit + 8 * p;
    const int nbits = std::min(8, end_bit - sh);
    cudaError_t e = run_pass<uint64_t, 0>(ci, cv, ko, vo, (uint32_t)n, sh, nbits,
                                          base + 256 * p, region + (size_t)p * nb * 256, ctrs + p, nullptr, nullptr,
                                          0, 0, st);
    if (e != cudaSuccess) return check_cuda(ctx, e, "sort pass u64");
    ci = ko;
    cv = vo;
  }
  return GSR_OK;
}

}  // namespace gsr

using namespace gsr;

extern "C" gsr_status gsr_sort_pairs_u64(gsr_ctx* ctx, const uint64_t* keys_in, const uint32_t* vals_in,
                                         uint64_t* keys_out, uint32_t* vals_out, int64_t n, int32_t begin_bit,
                                         int32_t end_bit, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (n < 0 || n >= (1ll << 31)) return set_err(ctx, GSR_EINVAL, "gsr_sort_pairs_u64: n out of range");
  if (begin_bit < 0 || end_bit > 64 || begin_bit >= end_bit)
    return set_err(ctx, GSR_EINVAL, "gsr_sort_pairs_u64: bad bit range");
  if (n > 0 && (!keys_in || !vals_in || !keys_out || !vals_out))
    return set_err(ctx, GSR_EINVAL, "gsr_sort_pairs_u64: NULL pointer");
  if (n == 0) return GSR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int passes = (end_bit - begin_bit + 7) / 8;
  const size_t nb = (size_t)((n + pass_tile<uint64_t>() - 1) / pass_tile<uint64_t>());
  void *kt, *vt, *hs, *lb;
  gsr_status s;
  if ((s = ensure(ctx, S_SORTK, n * 8, &kt)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_SORTV, n * 4, &vt)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_HIST, 2 * 8 * 256 * 4, &hs)) != GSR_OK) return s;
  const size_t lb_bytes = align_up(passes * nb * 256 * 4) + 64 * 4;
  if ((s = ensure(ctx, S_LOOKBACK, lb_bytes, &lb)) != GSR_OK) return s;
  uint32_t* hist = (uint32_t*)hs;
  uint32_t* base = hist + 8 * 256;
  uint32_t* look = (uint32_t*)lb;
  uint32_t* ctrs = (uint32_t*)((char*)lb + align_up(passes * nb * 256 * 4));
  if ((s = check_cuda(ctx, cudaMemsetAsync(hist, 0, 8 * 256 * 4, st), "memset")) != GSR_OK) return s;
  if ((s = check_cuda(ctx, cudaMemsetAsync(lb, 0, lb_bytes, st), "memset")) != GSR_OK) return s;
  const int hb = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 8);
  StageScope scope(ctx, GSR_STAGE_SORT_U64, st);
  account(ctx, GSR_STAGE_SORT_U64, 2 + passes, 8.0 * n + 24.0 * passes * n);
  hist_u64<<<hb, 256, 0, st>>>(keys_in, n, begin_bit, passes, end_bit, hist);
  scan_hist<<<1, 256, 0, st>>>(hist, base, passes);
  if ((s = check_cuda(ctx, cudaGetLastError(), "hist")) != GSR_OK) return s;
  return sort_u64_passes(ctx, keys_in, vals_in, keys_out, vals_out, (uint64_t*)kt, (uint32_t*)vt, n, begin_bit,
                         end_bit, base, look, ctrs, st);
}

struct CachedOrder {  // NEXT-2b: device visiting table [V][n_seg] + cache
  const OrderSeg* segs;
  int n_seg;
  const uint32_t* cache;
};

static gsr_status bin_sort_impl(gsr_ctx* ctx, const uint32_t* bin_rec, int64_t n, const gsr_camera* cams,
                                int32_t n_views, uint64_t* keys, uint32_t* vals, int64_t capacity, int64_t* n_keys,
                                uint32_t* ranges, uint64_t* keys_unsorted, uint32_t* vals_unsorted,
                                const CachedOrder* co, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!bin_rec || !cams || !vals || !n_keys || !ranges)
    return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: NULL required pointer");
  if (n < 0 || n_views <= 0 || n_views > GSR_MAX_VIEWS || capacity < 0)
    return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: bad n / n_views / capacity");
  if ((keys_unsorted == nullptr) != (vals_unsorted == nullptr))
    return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: keys_unsorted and vals_unsorted go together");
  const int W = cams[0].width, H = cams[0].height;
  for (int c = 0; c < n_views; ++c)
    if (cams[c].width != W || cams[c].height != H || W <= 0 || H <= 0)
      return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: mixed or non-positive resolutions in a batch");
  const uint32_t gx = (W + kTile - 1) / kTile, gy = (H + kTile - 1) / kTile;
  const uint64_t tpv = (uint64_t)gx * gy;
  const uint64_t T = tpv * (uint64_t)n_views;
  if (T >= (1ull << 32)) return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: V*tiles >= 2^32");
  const int64_t M = n * (int64_t)n_views;
  if (M >= (1ll << 30)) return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: V*n >= 2^30");
  cudaStream_t st = (cudaStream_t)stream;
  gsr_status s;

  const uint4* p_span = reinterpret_cast<const uint4*>(bin_rec);  // [M][2] span records
  const uint32_t* p_depth = bin_rec + 8 * M;
  const uint32_t* p_nt = bin_rec + 9 * M;

  const int vbits = bits_for((uint64_t)n_views);
  const int tbits = bits_for(T);
  const int tpasses = std::max(1, (tbits + 7) / 8);       // tile sort passes
  if (tpasses > 4) return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: batch too large");
  // depth keys: 32-bit (view << dshift | depth - dbase) unless they do not fit
  const int dshift = 32 - std::max(vbits, 1);
  float zmin = cams[0].znear;
  for (int c = 1; c < n_views; ++c) zmin = std::min(zmin, cams[c].znear);
  uint32_t dbase_bits;
  std::memcpy(&dbase_bits, &zmin, 4);
  bool wide = ctx->depth_keys64 || vbits > 8;
  const int cshift = 26;  // cached order: view << 26 (<= 64 views), no depth bits

  // ---- K2: compact + totals ----
  void *dka, *dkb, *dva, *dvb, *hs, *lb, *tot, *eo = nullptr;
  const size_t Mz = (size_t)std::max<int64_t>(M, 1);
  if ((s = ensure(ctx, S_DKEY_A, Mz * 8, &dka)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_DKEY_B, Mz * 8, &dkb)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_DVAL_A, Mz * 4, &dva)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_DVAL_B, Mz * 4, &dvb)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_HIST, 4 * 8 * 256 * 4, &hs)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_TOTALS, 64, &tot)) != GSR_OK) return s;
  if (keys_unsorted && (s = ensure(ctx, S_EMITOFF, Mz * 4, &eo)) != GSR_OK) return s;
  uint32_t* dhist = (uint32_t*)hs;          // [5][256]
  uint32_t* dbase = dhist + 8 * 256;        // [5][256]
  uint32_t* thist = dhist + 16 * 256;       // [4][256]
  uint32_t* tbase = dhist + 24 * 256;       // [4][256]
  const size_t nb2 = (size_t)((M + K2_TILE - 1) / K2_TILE);
  const size_t lb1 = align_up(2 * std::max<size_t>(nb2, 1) * 8) + 256;
  if ((s = ensure(ctx, S_LOOKBACK, lb1, &lb)) != GSR_OK) return s;
  uint64_t* lbv = (uint64_t*)lb;
  uint64_t* lbk = lbv + std::max<size_t>(nb2, 1);
  uint32_t* ctr2 = (uint32_t*)((char*)lb + align_up(2 * std::max<size_t>(nb2, 1) * 8));
  uint64_t* hp = (uint64_t*)ctx->host_pinned;
  int dpasses = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    dpasses = wide ? (32 + vbits + 7) / 8 : 4;
    if ((s = check_cuda(ctx, cudaMemsetAsync(lb, 0, lb1, st), "memset lb")) != GSR_OK) return s;
    if ((s = check_cuda(ctx, cudaMemsetAsync(dhist, 0, 8 * 256 * 4, st), "memset hist")) != GSR_OK) return s;
    if ((s = check_cuda(ctx, cudaMemsetAsync(tot, 0, 64, st), "memset tot")) != GSR_OK) return s;
    const int sp2 = stage_begin(ctx, GSR_STAGE_COMPACT, st);
    if (M > 0 && !co && wide)
      k2_compact<uint64_t><<<(unsigned)nb2, 256, 0, st>>>(p_depth, p_nt, M, n, (uint64_t*)dka, (uint32_t*)dva,
                                                          (uint32_t*)eo, lbv, lbk, ctr2, (uint64_t*)tot, dhist,
                                                          dpasses, 32, 0u);
    if (M > 0 && !co && !wide)
      k2_compact<uint32_t><<<(unsigned)nb2, 256, 0, st>>>(p_depth, p_nt, M, n, (uint32_t*)dka, (uint32_t*)dva,
                                                          (uint32_t*)eo, lbv, lbk, ctr2, (uint64_t*)tot, dhist,
                                                          dpasses, dshift, dbase_bits);
    if (M > 0 && co)
      k2c_compact<<<(unsigned)nb2, 256, 0, st>>>(co->segs, co->n_seg, co->cache, p_nt, M, n, (uint32_t*)dka,
                                                 (uint32_t*)dva, lbv, lbk, ctr2, (uint64_t*)tot, cshift);
    stage_end(ctx, sp2, st);
    if ((s = check_cuda(ctx, cudaGetLastError(), "k2_compact")) != GSR_OK) return s;
    if ((s = check_cuda(ctx, cudaMemcpyAsync(hp, tot, 24, cudaMemcpyDeviceToHost, st), "readback")) != GSR_OK)
      return s;
    if ((s = check_cuda(ctx, cudaStreamSynchronize(st), "sync")) != GSR_OK) return s;
    if (co || wide || hp[2] == 0) break;
    wide = true;  // a depth offset did not fit in 32 - vbits bits: redo with 64-bit keys
  }
  const int64_t nvis = (int64_t)hp[0];
  const int64_t K = (int64_t)hp[1];
  *n_keys = K;
  ctx->last_nvis = nvis;
  ctx->last_keys = K;
  // algorithmic bytes: K2 reads n_tiles of every pair and the depth of
  // the visible ones, writes 12 B per visible pair; K1's 48-B render records of
  // the visible pairs are attributed to the projection stage.
  account(ctx, GSR_STAGE_COMPACT, M > 0 ? 1 : 0,
          (co ? 8.0 : 4.0) * M + (co ? 0.0 : 4.0) * nvis + (wide && !co ? 12.0 : 8.0) * nvis);
  account(ctx, GSR_STAGE_PROJECT, 0, 80.0 * nvis);
  if (K > capacity) return set_err(ctx, GSR_ECAPACITY, "gsr_bin_sort: capacity too small (n_keys = required)");
  if (K >= (1ll << 31)) return set_err(ctx, GSR_EINVAL, "gsr_bin_sort: K >= 2^31 keys in one batch");

  if (K == 0) {
    if ((s = check_cuda(ctx, cudaMemsetAsync(ranges, 0, T * 8, st), "memset ranges")) != GSR_OK) return s;
    return GSR_OK;
  }

  // ---- scratch for the rest ----
  void *tka, *tkb, *tva, *tvb, *cnt;
  if ((s = ensure(ctx, S_TKEY_A, K * 4, &tka)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_TKEY_B, K * 4, &tkb)) != GSR_OK) return s;
  // two u32 arrays; the second starts 256-B aligned (TMA bulk copies need 16-B aligned sources)
  if ((s = ensure(ctx, S_TVAL_A, 2 * align_up(K * 4), &tva)) != GSR_OK) return s;
  tvb = (char*)tva + align_up(K * 4);
  if ((s = ensure(ctx, S_COUNTS, T * 4, &cnt)) != GSR_OK) return s;
  const size_t dtile = wide ? pass_tile<uint64_t>() : pass_tile<uint32_t>();
  const size_t ttile = pass_tile<uint32_t>();
  const size_t nbd = (size_t)((nvis + dtile - 1) / dtile);
  const size_t nb3 = (size_t)((nvis + K3_TILE - 1) / K3_TILE);
  const size_t nbt = (size_t)((K + ttile - 1) / ttile);
  const size_t o_d = 0;
  const size_t o_3 = align_up(o_d + dpasses * nbd * 256 * 4);
  const size_t o_t = align_up(o_3 + nb3 * 8);
  const size_t nb5 = (size_t)((T + K5_TILE - 1) / K5_TILE);
  const size_t o_5 = align_up(o_t + tpasses * nbt * 256 * 4);
  const size_t o_c = align_up(o_5 + nb5 * 8);
  const size_t lb2 = o_c + 64 * 4;
  // K2's look-back words are dead now (the sync above ordered them): reuse the slot.
  if ((s = ensure(ctx, S_LOOKBACK, lb2, &lb)) != GSR_OK) return s;
  if ((s = check_cuda(ctx, cudaMemsetAsync(lb, 0, lb2, st), "memset lb2")) != GSR_OK) return s;
  if ((s = check_cuda(ctx, cudaMemsetAsync(cnt, 0, T * 4, st), "memset counts")) != GSR_OK) return s;
  uint32_t* lbd = (uint32_t*)((char*)lb + o_d);
  uint64_t* lb3 = (uint64_t*)((char*)lb + o_3);
  uint32_t* lbt = (uint32_t*)((char*)lb + o_t);
  uint64_t* lb5 = (uint64_t*)((char*)lb + o_5);
  uint32_t* ctrs = (uint32_t*)((char*)lb + o_c);  // [0..4] depth, [5] k3, [6..9] tile, [10] k5

  // ---- K4a: depth sort of the visible pairs (skipped in the cached order) ----
  const void* ck = dka;
  const uint32_t* cvv = (const uint32_t*)dva;
  if (!co) {
    int spd = stage_begin(ctx, GSR_STAGE_DEPTH_SORT, st);
    scan_hist<<<1, 256, 0, st>>>(dhist, dbase, dpasses);
    const int kbits = wide ? 32 + vbits : 32;
    for (int p = 0; p < dpasses; ++p) {
      void* ko = (p % 2 == 0) ? dkb : dka;
      uint32_t* vo = (p % 2 == 0) ? (uint32_t*)dvb : (uint32_t*)dva;
      const int sh = 8 * p;
      cudaError_t e = wide ? run_pass<uint64_t, 0>((const uint64_t*)ck, cvv, (uint64_t*)ko, vo,
                                                   (uint32_t)nvis, sh, std::min(8, kbits - sh), dbase + 256 * p,
                                                   lbd + (size_t)p * nbd * 256, ctrs + p, nullptr, nullptr, 0, 0, st)
                           : run_pass<uint32_t, 0>((const uint32_t*)ck, cvv, (uint32_t*)ko, vo,
                                                   (uint32_t)nvis, sh, 8, dbase + 256 * p,
                                                   lbd + (size_t)p * nbd * 256, ctrs + p, nullptr, nullptr, 0, 0, st);
      if ((s = check_cuda(ctx, e, "depth sort pass")) != GSR_OK) return s;
      ck = ko;
      cvv = vo;
    }
    stage_end(ctx, spd, st);
    account(ctx, GSR_STAGE_DEPTH_SORT, 1 + dpasses, (wide ? 24.0 : 16.0) * dpasses * nvis);
    if ((s = check_cuda(ctx, cudaGetLastError(), "depth sort")) != GSR_OK) return s;
  }

  // K4c (counting scatter) unless the tile count is too large or the radix
  // tile sort is forced; its keys travel packed (tile << gbits | g, one
  // 4-B word per key instead of two) when both fit in 32 bits
  const bool use_cs = ctx->tile_sort_mode != 2 && tpv <= (uint64_t)CS_MAX_TPV;
  const int gbits = (use_cs && ctx->pack_tile_keys && bits_for(tpv) + std::max(1, bits_for(n)) <= 32)
                        ? std::max(1, bits_for(n)) : 0;

  // ---- K3: emission + counts ----
  int sp = stage_begin(ctx, GSR_STAGE_EMIT, st);
  const int bins = tpv <= 12288 ? (int)tpv : 0;  // <= 48 KB of dynamic shared memory (opt-in above 48 KB total)
  if (wide && !co) {
    auto k3 = gbits ? k3_emit<uint64_t, true> : k3_emit<uint64_t, false>;
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, bins * 4);
    k3<<<(unsigned)nb3, 256, bins * 4, st>>>((const uint64_t*)ck, cvv, nvis, p_span, n, gx, (uint32_t)tpv, W,
                                             (uint32_t*)tka, (uint32_t*)tva, (uint32_t*)cnt, lb3, ctrs + 5, bins,
                                             32, gbits, (uint64_t)K, T);
  } else {
    auto k3 = gbits ? k3_emit<uint32_t, true> : k3_emit<uint32_t, false>;
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, bins * 4);
    k3<<<(unsigned)nb3, 256, bins * 4, st>>>((const uint32_t*)ck, cvv, nvis, p_span, n, gx, (uint32_t)tpv, W,
                                             (uint32_t*)tka, (uint32_t*)tva, (uint32_t*)cnt, lb3, ctrs + 5, bins,
                                             co ? cshift : dshift, gbits, (uint64_t)K, T);
  }
  stage_end(ctx, sp, st);
  account(ctx, GSR_STAGE_EMIT, 1, 44.0 * nvis + (gbits ? 4.0 : 8.0) * K + 4.0 * T);
  if ((s = check_cuda(ctx, cudaGetLastError(), "k3_emit")) != GSR_OK) return s;

  // ---- K5: ranges + tile-sort histograms ----
  sp = stage_begin(ctx, GSR_STAGE_RANGES, st);
  // (the K4b radix passes also need the tile-digit histograms: one block)
  if (use_cs)
    k5_scan<<<(unsigned)nb5, 256, 0, st>>>((const uint32_t*)cnt, (int64_t)T, (uint2*)ranges, lb5, ctrs + 10);
  else
    k5_ranges<<<1, 1024, 0, st>>>((const uint32_t*)cnt, (int64_t)T, (uint2*)ranges, tpasses, thist, tbase);
  stage_end(ctx, sp, st);
  account(ctx, GSR_STAGE_RANGES, 1, 12.0 * T);
  if ((s = check_cuda(ctx, cudaGetLastError(), "k5_ranges")) != GSR_OK) return s;

  // ---- K4b / K4c: tile sort ----
  // K4c (default, up to CS_MAX_TPV tiles per view: cs_hist keeps one view's
  // counters in 48 KB of shared memory); tile counts above CS_AUTO_TPV are
  // split into slices so 8 warps' scatter counters still fit twice per SM
  // (measured: c3 2,500 tiles 1.09 -> 0.79 ms per batch; c4 8,160 tiles in 2
  // slices 804 vs 799 views/s for the radix passes; unsliced with 4 warps 609).
  // GSR_TSORT=radix forces the two onesweep passes.
  if (use_cs) {
    // K4c counting scatter (default)
    const uint32_t ch = (uint32_t)CS_CHUNK;
    const uint64_t nchunks_max = (uint64_t)(K + ch - 1) / ch + (uint64_t)n_views;
    void *hm, *meta;
    if ((s = ensure(ctx, S_CSH, nchunks_max * tpv * 4, &hm)) != GSR_OK) return s;
    if ((s = ensure(ctx, S_CSMETA, 2 * (n_views + 1) * 4, &meta)) != GSR_OK) return s;
    const int nslice = (int)((tpv + CS_AUTO_TPV - 1) / CS_AUTO_TPV);
    const uint32_t tslice = (uint32_t)((tpv + nslice - 1) / nslice);
    const size_t smem = (size_t)((tslice + 7) & ~7u) * (8 + 2 * 8);
    sp = stage_begin(ctx, GSR_STAGE_TILE_SORT, st);
    cs_meta<<<1, 64, 0, st>>>((const uint2*)ranges, n_views, (uint32_t)tpv, (uint32_t)K, (uint32_t*)meta, ch);
    cs_hist<<<(unsigned)nchunks_max, 256, tpv * 4, st>>>((const uint32_t*)tka, (const uint32_t*)meta, n_views,
                                                          (uint32_t)tpv, (uint32_t*)hm, gbits, ch);
    cs_scan<<<(unsigned)((T + 255) / 256), 256, 0, st>>>((const uint2*)ranges, (const uint32_t*)meta, n_views,
                                                         (uint32_t)tpv, (uint32_t*)hm);
    const int dbits = std::max(1, bits_for(tslice));
    // compile-time digit widths (8 / 10 / 12 / 14 bits; CS_MAX_TPV needs at most 14)
    auto scat = gbits ? (dbits <= 8 ? cs_scatter<8, true, 8> : dbits <= 10 ? cs_scatter<8, true, 10>
                         : dbits <= 12 ? cs_scatter<8, true, 12> : dbits <= 14 ? cs_scatter<8, true, 14>
                         : cs_scatter<8, true>)
                      : (dbits <= 8 ? cs_scatter<8, false, 8> : dbits <= 10 ? cs_scatter<8, false, 10>
                         : dbits <= 12 ? cs_scatter<8, false, 12> : dbits <= 14 ? cs_scatter<8, false, 14>
                         : cs_scatter<8, false>);
    cudaFuncSetAttribute(scat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    scat<<<(unsigned)(nchunks_max * nslice), 256, smem, st>>>(
        (const uint32_t*)tka, (const uint32_t*)tva, (const uint32_t*)meta, n_views, (uint32_t)tpv, dbits, tslice,
        nslice, (const uint32_t*)hm, vals, keys, p_depth, n, gbits, ch);
    stage_end(ctx, sp, st);
    // hist reads 4 B/key; scatter reads 8 B/key (4 B packed) and writes the
    // 4-B values (+ 8-B keys when asked); the chunk x tile matrix is written,
    // scanned in place and read once
    const double hbytes = (double)(K + ch - 1) / ch * (double)tpv * 4.0;
    account(ctx, GSR_STAGE_TILE_SORT, 4, ((gbits ? 12.0 : 16.0) + (keys ? 8.0 : 0.0)) * K + 4.0 * hbytes);
    if ((s = check_cuda(ctx, cudaGetLastError(), "tile counting scatter")) != GSR_OK) return s;
  } else {
  sp = stage_begin(ctx, GSR_STAGE_TILE_SORT, st);
  const uint32_t* tk = (const uint32_t*)tka;
  const uint32_t* tv = (const uint32_t*)tva;
  for (int p = 0; p < tpasses; ++p) {
    const int sh = 8 * p;
    const int nbits = std::max(1, std::min(8, tbits - sh));
    uint32_t* lbp = lbt + (size_t)p * nbt * 256;
    cudaError_t e;
    if (p == tpasses - 1) {
      e = run_pass<uint32_t, 1>(tk, tv, nullptr, vals, (uint32_t)K, sh, nbits, tbase + 256 * p, lbp, ctrs + 6 + p,
                                keys, p_depth, (uint32_t)tpv, n, st);
    } else {
      uint32_t* ko = (p % 2 == 0) ? (uint32_t*)tkb : (uint32_t*)tka;
      uint32_t* vo = (p % 2 == 0) ? (uint32_t*)tvb : (uint32_t*)tva;
      e = run_pass<uint32_t, 0>(tk, tv, ko, vo, (uint32_t)K, sh, nbits, tbase + 256 * p, lbp, ctrs + 6 + p, nullptr,
                                nullptr, 0, 0, st);
      tk = ko;
      tv = vo;
    }
    if ((s = check_cuda(ctx, e, "tile sort pass")) != GSR_OK) return s;
  }
  stage_end(ctx, sp, st);
  // each pass reads 8 B/key; intermediate passes write 8 B/key, the last writes
  // the 4-B values (+ 8-B keys when asked)
  account(ctx, GSR_STAGE_TILE_SORT, tpasses,
          16.0 * (tpasses - 1) * K + (12.0 + (keys ? 8.0 : 0.0)) * K);
  if ((s = check_cuda(ctx, cudaGetLastError(), "tile sort")) != GSR_OK) return s;

  }

  // ---- optional O2 emission-order list ----
  if (keys_unsorted) {
    account(ctx, GSR_STAGE_EMIT, 1, 16.0 * M + 12.0 * K);
    k_emit_o2<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(p_depth, p_span, p_nt, (const uint32_t*)eo, M, n, gx,
                                                           (uint32_t)tpv, W, keys_unsorted, vals_unsorted);
    if ((s = check_cuda(ctx, cudaGetLastError(), "emit_o2")) != GSR_OK) return s;
  }
  return GSR_OK;
}

extern "C" gsr_status gsr_bin_sort(gsr_ctx* ctx, const uint32_t* bin_rec, int64_t n, const gsr_camera* cams,
                                   int32_t n_views, uint64_t* keys, uint32_t* vals, int64_t capacity,
                                   int64_t* n_keys, uint32_t* ranges, uint64_t* keys_unsorted,
                                   uint32_t* vals_unsorted, void* stream) {
  return bin_sort_impl(ctx, bin_rec, n, cams, n_views, keys, vals, capacity, n_keys, ranges, keys_unsorted,
                       vals_unsorted, nullptr, stream);
}

// ---- NEXT-2b: cached view-direction orderings ----
static gsr_status check_tiles(gsr_ctx* ctx, const int64_t* tile_start, int32_t n_tiles, const int32_t* bins,
                              int64_t n, const char* who) {
  if (!tile_start || !bins || n_tiles <= 0 || n_tiles > 4096)
    return set_err(ctx, GSR_EINVAL, std::string(who) + ": bad tile table");
  if (tile_start[0] != 0 || tile_start[n_tiles] != n)
    return set_err(ctx, GSR_EINVAL, std::string(who) + ": tile ranges must cover [0, n)");
  for (int t = 0; t < n_tiles; ++t) {
    if (tile_start[t + 1] < tile_start[t]) return set_err(ctx, GSR_EINVAL, std::string(who) + ": tile ranges");
    if (bins[t] < 1 || bins[t] > 64) return set_err(ctx, GSR_EINVAL, std::string(who) + ": bins in [1, 64]");
  }
  return GSR_OK;
}

extern "C" int64_t gsr_order_cache_size(const int64_t* tile_start, int32_t n_tiles, const int32_t* bins) {
  if (!tile_start || !bins || n_tiles <= 0) return 0;
  int64_t s = 0;
  for (int t = 0; t < n_tiles; ++t) s += (int64_t)bins[t] * (tile_start[t + 1] - tile_start[t]);
  return s;
}

extern "C" gsr_status gsr_build_order_cache(gsr_ctx* ctx, const gsr_gaussians* G, const int64_t* tile_start,
                                            int32_t n_tiles, const int32_t* bins, uint32_t* cache, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!G || !cache) return set_err(ctx, GSR_EINVAL, "gsr_build_order_cache: NULL required pointer");
  gsr_status s;
  if ((s = check_tiles(ctx, tile_start, n_tiles, bins, G->n, "gsr_build_order_cache")) != GSR_OK) return s;
  std::vector<CacheSeg> segs;
  uint64_t out = 0;
  uint32_t maxlen = 0;
  for (int t = 0; t < n_tiles; ++t) {
    const uint32_t len = (uint32_t)(tile_start[t + 1] - tile_start[t]);
    maxlen = std::max(maxlen, len);
    for (int k = 0; k < bins[t]; ++k) {
      const double a = 2.0 * M_PI * k / bins[t];
      segs.push_back(CacheSeg{out, (uint32_t)tile_start[t], len, (float)std::cos(a), (float)std::sin(a)});
      out += len;
    }
  }
  const int64_t N = (int64_t)out;
  if (N == 0) return GSR_OK;
  if (N >= (1ll << 31)) return set_err(ctx, GSR_EINVAL, "gsr_build_order_cache: cache too large");
  cudaStream_t st = (cudaStream_t)stream;
  // the bin-sort scratch slots hold the sort input / key output (the utility
  // sort's own temporaries live in S_SORTK / S_SORTV)
  void *tab, *k0, *k1, *v0;
  const size_t tb = segs.size() * sizeof(CacheSeg);
  if ((s = ensure(ctx, S_SELECT2, tb, &tab)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_DKEY_A, (size_t)N * 8, &k0)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_DKEY_B, (size_t)N * 8, &k1)) != GSR_OK) return s;
  if ((s = ensure(ctx, S_DVAL_A, (size_t)N * 4, &v0)) != GSR_OK) return s;
  if ((s = check_cuda(ctx, cudaMemcpyAsync(tab, segs.data(), tb, cudaMemcpyHostToDevice, st), "segs")) != GSR_OK)
    return s;
  uint64_t* keys = (uint64_t*)k0;
  uint64_t* keys_out = (uint64_t*)k1;
  uint32_t* vals = (uint32_t*)v0;
  const dim3 grid((unsigned)std::min<uint32_t>((maxlen + 255) / 256, 1024), (unsigned)segs.size());
  kc_keys<<<grid, 256, 0, st>>>((const CacheSeg*)tab, reinterpret_cast<const float4*>(G->pos_opacity), keys, vals);
  if ((s = check_cuda(ctx, cudaGetLastError(), "kc_keys")) != GSR_OK) return s;
  // stable sort by (segment, key): the sorted values are the cache
  const int end_bit = 32 + std::max(1, bits_for(segs.size()));
  return gsr_sort_pairs_u64(ctx, keys, vals, keys_out, cache, N, 0, end_bit, stream);
}

// NEXT-2b cache policy (§3.5 "tiles whose uncertainty
// exceeds threshold tau retain a larger set of cached orderings", tau = 0.6
// §3.6): per tile the mean per-Gaussian uncertainty (double, fixed-order
// block sum), hot_bins if it exceeds tau, else base_bins.
__global__ void __launch_bounds__(256) k_cache_bins(const float4* __restrict__ su, const int64_t* __restrict__ start,
                                                    float tau, int32_t base_bins, int32_t hot_bins,
                                                    int32_t* __restrict__ bins) {
  __shared__ double s_w[8];
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t a = start[t], b = start[t + 1];
  double acc = 0.0;
  for (int64_t i = a + tid; i < b; i += 256) acc += (double)__ldg(&su[i].w);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
  if (lane == 0) s_w[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < 8; ++w) sum += s_w[w];
    const double mean = b > a ? sum / (double)(b - a) : 0.0;
    bins[t] = mean > (double)tau ? hot_bins : base_bins;
  }
}

extern "C" gsr_status gsr_bin_sort_cached(gsr_ctx* ctx, const uint32_t* bin_rec, int64_t n, const gsr_camera* cams,
                                          int32_t n_views, const uint32_t* cache, const int64_t* tile_start,
                                          int32_t n_tiles, const int32_t* bins, const double* centres,
                                          uint64_t* keys, uint32_t* vals, int64_t capacity, int64_t* n_keys,
                                          uint32_t* ranges, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!cache || !centres || !cams) return set_err(ctx, GSR_EINVAL, "gsr_bin_sort_cached: NULL required pointer");
  if (n_views <= 0 || n_views > GSR_MAX_VIEWS) return set_err(ctx, GSR_EINVAL, "gsr_bin_sort_cached: bad n_views");
  gsr_status s;
  if ((s = check_tiles(ctx, tile_start, n_tiles, bins, n, "gsr_bin_sort_cached")) != GSR_OK) return s;
  // per view: the chosen bin of every tile and the tiles' visiting order (host, double)
  std::vector<uint64_t> base(n_tiles);
  uint64_t off = 0;
  for (int t = 0; t < n_tiles; ++t) {
    base[t] = off;
    off += (uint64_t)bins[t] * (uint64_t)(tile_start[t + 1] - tile_start[t]);
  }
  std::vector<OrderSeg> segs((size_t)n_views * n_tiles);
  std::vector<int> order(n_tiles);
  std::vector<double> depth(n_tiles);
  for (int v = 0; v < n_views; ++v) {
    const gsr_camera& c = cams[v];
    const double f[3] = {c.R[6], c.R[7], c.R[8]};
    const double eye[3] = {c.campos[0], c.campos[1], c.campos[2]};
    double h0 = f[0], h1 = f[2];
    const double hn = std::max(std::sqrt(h0 * h0 + h1 * h1), 1e-30);
    h0 /= hn;
    h1 /= hn;
    for (int t = 0; t < n_tiles; ++t) {
      depth[t] = ((centres[3 * t] - eye[0]) * f[0] + (centres[3 * t + 1] - eye[1]) * f[1]) +
                 (centres[3 * t + 2] - eye[2]) * f[2];
      order[t] = t;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return depth[a] < depth[b]; });
    uint32_t pos = 0;
    for (int i = 0; i < n_tiles; ++i) {
      const int t = order[i];
      int best = 0;
      double bd = -1e300;
      for (int k = 0; k < bins[t]; ++k) {
        const double a = 2.0 * M_PI * k / bins[t];
        const double d = h0 * std::cos(a) + h1 * std::sin(a);
        if (d > bd) {
          bd = d;
          best = k;
        }
      }
      const uint32_t len = (uint32_t)(tile_start[t + 1] - tile_start[t]);
      segs[(size_t)v * n_tiles + i] = OrderSeg{base[t] + (uint64_t)best * len, pos, len};
      pos += len;
    }
  }
  void* tab;
  const size_t tb = segs.size() * sizeof(OrderSeg);
  if ((s = ensure(ctx, S_SELECT2, tb, &tab)) != GSR_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = check_cuda(ctx, cudaMemcpyAsync(tab, segs.data(), tb, cudaMemcpyHostToDevice, st), "order table")) !=
      GSR_OK)
    return s;
  CachedOrder co{(const OrderSeg*)tab, n_tiles, cache};
  return bin_sort_impl(ctx, bin_rec, n, cams, n_views, keys, vals, capacity, n_keys, ranges, nullptr, nullptr, &co,
                       stream);
}

extern "C" gsr_status gsr_order_cache_bins(gsr_ctx* ctx, const gsr_gaussians* G, const int64_t* tile_start,
                                           int32_t n_tiles, float tau, int32_t base_bins, int32_t hot_bins,
                                           int32_t* bins, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!G || !tile_start || !bins || n_tiles <= 0 || n_tiles > 4096)
    return set_err(ctx, GSR_EINVAL, "gsr_order_cache_bins: NULL pointer or bad n_tiles");
  if (base_bins < 1 || base_bins > 64 || hot_bins < 1 || hot_bins > 64)
    return set_err(ctx, GSR_EINVAL, "gsr_order_cache_bins: bins in [1, 64]");
  if (tile_start[0] != 0 || tile_start[n_tiles] != G->n)
    return set_err(ctx, GSR_EINVAL, "gsr_order_cache_bins: tile ranges must cover [0, n)");
  for (int t = 0; t < n_tiles; ++t)
    if (tile_start[t + 1] < tile_start[t]) return set_err(ctx, GSR_EINVAL, "gsr_order_cache_bins: tile ranges");
  cudaStream_t st = (cudaStream_t)stream;
  gsr_status s;
  void* tab;
  const size_t tb = (size_t)(n_tiles + 1) * 8 + (size_t)n_tiles * 4;
  if ((s = ensure(ctx, S_SELECT2, tb, &tab)) != GSR_OK) return s;
  int64_t* d_start = (int64_t*)tab;
  int32_t* d_bins = (int32_t*)((char*)tab + (size_t)(n_tiles + 1) * 8);
  if ((s = check_cuda(ctx, cudaMemcpyAsync(d_start, tile_start, (size_t)(n_tiles + 1) * 8, cudaMemcpyHostToDevice, st),
                      "tile table")) != GSR_OK)
    return s;
  k_cache_bins<<<n_tiles, 256, 0, st>>>(reinterpret_cast<const float4*>(G->scale_unc), d_start, tau, base_bins,
                                         hot_bins, d_bins);
  if ((s = check_cuda(ctx, cudaGetLastError(), "k_cache_bins")) != GSR_OK) return s;
  if ((s = check_cuda(ctx, cudaMemcpyAsync(bins, d_bins, (size_t)n_tiles * 4, cudaMemcpyDeviceToHost, st), "bins")) !=
      GSR_OK)
    return s;
  return check_cuda(ctx, cudaStreamSynchronize(st), "gsr_order_cache_bins sync");
}
