// gsr_internal.cuh -- shared declarations of libgsr (CUDA, sm_100a).
//
// Nothing here is shared with the CPU oracle (oracle/): the two implement the
// readings of DESIGN.md independently.
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/gsr.h"

// Device-side bounds checks of the debug build (build.py --debug ->
// libgsr_debug.so, GSR_LIB=...): compute-sanitizer is closed on the GPU
// pool, so every computed global index of the hot kernels is checked here
// and a violation traps with its location.
#ifdef GSR_DEBUG
#define GSR_DCHECK(cond)                                                          \
  do {                                                                            \
    if (!(cond)) {                                                                \
      printf("GSR_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
      __trap();                                                                   \
    }                                                                             \
  } while (0)
#else
#define GSR_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace gsr {

// ---- rasterizer constants (float32 hex in comments) ----
constexpr float kDilation = 0.3f;          // 0x3e99999a  EWA low-pass, px^2
constexpr float kAlphaMax = 0.99f;         // 0x3f7d70a4
constexpr float kTStop = 1e-4f;            // 0x38d1b717
constexpr uint32_t kAlphaMinBits = 0x3b808081u;  // 1/255
constexpr int kTile = GSR_TILE;

struct CamBatch {
  gsr_camera c[GSR_MAX_VIEWS];
};

struct LodParams {  // NEXT-2 LOD blending (gsr_lod), kernel parameter
  int on, levels;
  float delta;
  float D[7];
  const float* tile_level;
};

// exp(x) for x <= 0: Cody-Waite range reduction by ln2 (hi/lo), degree-7
// Taylor polynomial in Horner form, scale by 2^k built in the exponent field.
// Pure IEEE float ops -> bit-identical on any correctly rounding FPU.
__device__ __forceinline__ float exp_spec_core(float x) {  // x in [-80, 0]
  const float kf = rintf(x * __int_as_float(0x3fb8aa3b));
  float r = __fmaf_rn(kf, -__int_as_float(0x3f317200), x);
  r = __fmaf_rn(kf, -__int_as_float(0x35bfbe8e), r);
  float p = __int_as_float(0x39500d01);
  p = __fmaf_rn(p, r, __int_as_float(0x3ab60b61));
  p = __fmaf_rn(p, r, __int_as_float(0x3c088889));
  p = __fmaf_rn(p, r, __int_as_float(0x3d2aaaab));
  p = __fmaf_rn(p, r, __int_as_float(0x3e2aaaab));
  p = __fmaf_rn(p, r, __int_as_float(0x3f000000));
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  const int k = (int)kf;
  return p * __int_as_float((k + 127) << 23);
}
__device__ __forceinline__ float exp_spec(float x) { return x < -80.0f ? 0.0f : exp_spec_core(x); }
// The same function (bit for bit) with fewer issue slots off the FMA pipe:
// rint(y) for |y| < 2^22 as (y + 1.5 * 2^23) - 1.5 * 2^23 (round to nearest
// even, exactly what rintf does), and 2^k straight from the rounded sum's
// low bits: bits(y + 1.5 * 2^23) = 0x4B400000 + k, and 0x4B400000 << 23 == 0
// (mod 2^32), so (k + 127) << 23 == (bits << 23) + 0x3f800000.  c7 is the
// first Horner coefficient (0x39500d01) passed in a register the caller keeps
// live across its loop (FFMA takes one immediate).
__device__ __forceinline__ float exp_spec_core_fast(float x, float c7) {  // x in [-80, 0]
  const float t = __fadd_rn(__fmul_rn(x, __int_as_float(0x3fb8aa3b)), 12582912.0f);
  const float kf = __fsub_rn(t, 12582912.0f);
  float r = __fmaf_rn(kf, -__int_as_float(0x3f317200), x);
  r = __fmaf_rn(kf, -__int_as_float(0x35bfbe8e), r);
  float p = __fmaf_rn(c7, r, __int_as_float(0x3ab60b61));
  p = __fmaf_rn(p, r, __int_as_float(0x3c088889));
  p = __fmaf_rn(p, r, __int_as_float(0x3d2aaaab));
  p = __fmaf_rn(p, r, __int_as_float(0x3e2aaaab));
  p = __fmaf_rn(p, r, __int_as_float(0x3f000000));
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  return p * __int_as_float((int)((__float_as_uint(t) << 23) + 0x3f800000u));
}

// Packed FP32 (sm_100a FADD2 / FMUL2 / FFMA2): two IEEE round-to-nearest
// results per instruction, each identical to the scalar operation.  ptxas
// contracts a packed mul feeding a packed add into FFMA2 even under
// -fmad=false (and -Xptxas --fmad=false), so no packed product here ever
// feeds a packed add / sub.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f32x2 bc2(float v) { return pk2(v, v); }
__device__ __forceinline__ float lo2(f32x2 v) {
  float a;
  asm("mov.b64 {%0, _}, %1;" : "=f"(a) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi2(f32x2 v) {
  float b;
  asm("mov.b64 {_, %0}, %1;" : "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f32x2 fsub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// ---- tile spans (O1 steps 14-15) ----
// A Gaussian is listed in tile (tx, ty) iff the tile holds a pixel centre
// inside the x-extent, over the tile's pixel rows, of the ellipse q <= 11.1
// (> 3.33^2 > 2 ln 255: contains every alpha >= 1/255 pixel) widened by
// 1/16 px.  K1 stores the span parameters once per visible (view, g) in a
// 32-byte record; K1 (counting) and K3 (emitting) evaluate the same span
// function on the same floats, so n_tiles and the emitted keys agree exactly.
constexpr float kSpanT = 11.1f;      // 0x4131999a
constexpr float kSpanM = 0.0625f;    // 1/16 px
// span record [V*n][2] uint4: (u, v, p = b/c, h = det/c), (1/c, dys, py0 | py1 << 16, n_tiles)
__device__ __forceinline__ void row_span(float u, float v, float p, float h, float ic, float dys, uint32_t py0,
                                         uint32_t py1, uint32_t ty, int W, uint32_t& x0, uint32_t& x1) {
  const uint32_t ya = max(ty * 16u, py0), yb = min(ty * 16u + 15u, py1);
  const float dya = ((float)ya + 0.5f) - v;
  const float dyb = ((float)yb + 0.5f) - v;
  const float dr = fminf(fmaxf(dys, dya), dyb);
  const float dl = fminf(fmaxf(-dys, dya), dyb);
  const float R = ((u + p * dr) + sqrtf(fmaxf(0.0f, h * (kSpanT - (dr * dr) * ic)))) + kSpanM;
  const float L = ((u + p * dl) - sqrtf(fmaxf(0.0f, h * (kSpanT - (dl * dl) * ic)))) - kSpanM;
  const float fx0 = fmaxf(ceilf(L - 0.5f), 0.0f);
  const float fx1 = fminf(floorf(R - 0.5f), (float)(W - 1));
  if (fx0 <= fx1) {
    x0 = (uint32_t)fx0 >> 4;
    x1 = ((uint32_t)fx1 >> 4) + 1u;
  } else {
    x0 = 0u;
    x1 = 0u;
  }
}

// ---- context scratch ----
enum Slot {
  S_DKEY_A, S_DKEY_B, S_DVAL_A, S_DVAL_B,   // depth pre-sort (visible (view,g) pairs)
  S_TKEY_A, S_TKEY_B, S_TVAL_A,             // tile sort keys / payload ping-pong
  S_COUNTS,                                 // per (view,tile) key counts
  S_HIST,                                   // per-pass digit histograms + bases
  S_LOOKBACK,                               // decoupled look-back words
  S_EMITOFF,                                // emission offsets (parity output only)
  S_TOTALS,                                 // device totals (Nvis, K)
  S_SORTK, S_SORTV,                         // utility sort ping-pong
  S_SELECT,                                 // exclusion mask staging
  S_SELECT2,                                // NEXT-1 per-chunk partial sums
  S_GRAD2D,                                 // NEXT-3 per-(view, g) 2D gradients
  S_CSH, S_CSMETA,                          // K4c chunk x tile offsets, view / chunk table
  S_K6PART,                                 // K6 strip partial sums (four 16x4 strips per tile)
  S_OPTIM,                                  // NEXT-3 loss partial sums
  S_NSLOTS
};

}  // namespace gsr

struct gsr_ctx {
  int device = 0;
  std::string err;
  void* buf[gsr::S_NSLOTS] = {};
  size_t cap[gsr::S_NSLOTS] = {};
  void* host_pinned = nullptr;  // 4 KB pinned readback area
  int num_sms = 148;
  // diagnostics
  bool timing = false;
  struct Span {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<Span> spans;
  std::vector<cudaEvent_t> pool;
  double bytes[GSR_N_STAGES] = {};
  int64_t launches[GSR_N_STAGES] = {};
  int64_t last_nvis = 0, last_keys = 0;  // of the last gsr_bin_sort (byte accounting)
  bool depth_keys64 = false;  // force the 64-bit depth-sort keys (GSR_DKEY64=1)
  int bw_warps = 2;           // K6b warps per block: 2 (sub-tile blocks) or 8 (GSR_BWNW)
  int bw_reduce = 2;          // K6b warp reduction: 0 shuffle trees, 1 smem atomics, 2 butterfly (GSR_BWRED)
  int k6_persist = 0;         // K6 persistent grid: resident blocks per SM (gsr_set_composite_residency; 0 = one block per strip)
  int pack_tile_keys = 1;     // K3 -> K4c keys as one (tile << gbits | g) word when they fit (GSR_PACK=0: two planes)
  int tile_sort_mode = 0;     // 0 / 1: K4c counting scatter up to 12,288 tiles per view, 2: K4b radix (GSR_TSORT=radix)
};

namespace gsr {

// Every entry point runs on the context's device: libgsr links cudart
// statically, so it keeps its own per-thread current device, which another
// thread or a second context may have left elsewhere.  The caller's device
// is restored on return.
struct DeviceGuard {
  int prev = -1;
  bool restore = false;
  explicit DeviceGuard(const gsr_ctx* ctx) {
    if (ctx && cudaGetDevice(&prev) == cudaSuccess && prev != ctx->device)
      restore = cudaSetDevice(ctx->device) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (restore) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

gsr_status set_err(gsr_ctx* ctx, gsr_status st, const std::string& msg);
gsr_status check_cuda(gsr_ctx* ctx, cudaError_t e, const char* what);
gsr_status ensure(gsr_ctx* ctx, Slot s, size_t bytes, void** out);

// ---- diagnostics: stage spans (CUDA events) + launch / byte accounting ----
int stage_begin(gsr_ctx* ctx, int stage, cudaStream_t st);  // returns span id or -1
void stage_end(gsr_ctx* ctx, int span, cudaStream_t st);
inline void account(gsr_ctx* ctx, int stage, int64_t launches, double bytes) {
  ctx->launches[stage] += launches;
  ctx->bytes[stage] += bytes;
}
struct StageScope {
  gsr_ctx* ctx;
  int span;
  cudaStream_t st;
  StageScope(gsr_ctx* c, int stage, cudaStream_t s) : ctx(c), span(stage_begin(c, stage, s)), st(s) {}
  ~StageScope() { stage_end(ctx, span, st); }
};

// ---- launchers (each returns cudaGetLastError() of its launches) ----
cudaError_t launch_project(const gsr_gaussians& G, const CamBatch& cams, const LodParams& lod, int V, float* rec,
                           uint32_t* bin, cudaStream_t st);

// onesweep radix sort pieces (binsort.cu)
struct SortBufs {
  uint32_t* hist;      // [passes][256] histograms, then [passes][256] exclusive bases
  uint32_t* lookback;  // [passes][nblocks][256]
  uint32_t* counters;  // [passes] dynamic block ids
};

}  // namespace gsr
