// w2.cu -- NEXT-1: latent-space ensemble disagreement W2(Z), PAPER.md
// eq:w2_pixel (§3.3).  One 512-thread block per candidate view;
// threads stride over the H_z W_z latent locations; per location the C(M,2)
// sample pairs are evaluated exactly as the equation writes them
// (||mu_i - mu_j||^2 + sum_c (s2_i + s2_j - 2 sqrt(s2_i s2_j))), in float, and
// accumulated per thread in double; a fixed-order block reduction gives the
// view's spatial mean.  HBM-bound: every mean / variance is read once from
// DRAM (pair re-reads hit L1).
#include "gsr_internal.cuh"

namespace gsr {
namespace {

constexpr uint32_t FULL = 0xffffffffu;

__global__ void __launch_bounds__(512) k_w2(const float* __restrict__ mu, const float* __restrict__ s2, int M, int C,
                                            int64_t HW, float* __restrict__ scores, float* __restrict__ map) {
  __shared__ double s_w[16];
  const int v = blockIdx.x, tid = threadIdx.x;
  const size_t vo = (size_t)v * M * C * HW;
  const float* vm = mu + vo;
  const float* vs = s2 + vo;
  const float inv_pairs = 2.0f / (float)(M * (M - 1));
  double acc = 0.0;
  for (int64_t p = tid; p < HW; p += blockDim.x) {
    float sum = 0.0f;
    for (int i = 0; i < M; ++i)
      for (int j = i + 1; j < M; ++j) {
        float t = 0.0f;
        for (int c = 0; c < C; ++c) {
          const float d = __ldg(vm + ((size_t)i * C + c) * HW + p) - __ldg(vm + ((size_t)j * C + c) * HW + p);
          t = t + d * d;
        }
        for (int c = 0; c < C; ++c) {
          const float a = __ldg(vs + ((size_t)i * C + c) * HW + p), b = __ldg(vs + ((size_t)j * C + c) * HW + p);
          t = t + ((a + b) - 2.0f * sqrtf(a * b));
        }
        sum = sum + t;
      }
    if (map) map[(size_t)v * HW + p] = sum * inv_pairs;
    acc += (double)sum;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
  if ((tid & 31) == 0) s_w[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
    scores[v] = (float)(t / ((double)HW * (double)(M * (M - 1) / 2)));
  }
}

// Register-resident variant for compile-time (M, C): each (sample, channel)
// value of a location is loaded once (coalesced across the warp) and every
// pair is formed from registers -- the generic kernel re-issues the loads per
// pair and was load-issue bound (ncu-free estimate: 80 LDG per location).
template <int M, int C>
__global__ void __launch_bounds__(256) k_w2_t(const float* __restrict__ mu, const float* __restrict__ s2, int64_t HW,
                                              double* __restrict__ partial, float* __restrict__ map) {
  // grid (views, chunks): 256 threads x 4 locations per block, the block's
  // double partial sum goes to partial[view][chunk] (reduced by k_w2_fin in a
  // fixed order: deterministic).
  __shared__ double s_w[8];
  const int v = blockIdx.x, tid = threadIdx.x;
  const size_t vo = (size_t)v * M * C * HW;
  const float* vm = mu + vo;
  const float* vs = s2 + vo;
  constexpr int NP = M * (M - 1) / 2;
  const float inv_pairs = 1.0f / (float)NP;
  double acc = 0.0;
  const int64_t p0 = (int64_t)blockIdx.y * 1024;
  for (int64_t p = p0 + tid; p < HW && p < p0 + 1024; p += 256) {
    float a[M][C], s[M][C];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        a[m][ch] = __ldcs(vm + ((size_t)m * C + ch) * HW + p);
        s[m][ch] = __ldcs(vs + ((size_t)m * C + ch) * HW + p);
      }
    float sum = 0.0f;
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = i + 1; j < M; ++j) {
        float t = 0.0f;
#pragma unroll
        for (int ch = 0; ch < C; ++ch) {
          const float d = a[i][ch] - a[j][ch];
          t = t + d * d;
        }
#pragma unroll
        for (int ch = 0; ch < C; ++ch) t = t + ((s[i][ch] + s[j][ch]) - 2.0f * sqrtf(s[i][ch] * s[j][ch]));
        sum = sum + t;
      }
    if (map) map[(size_t)v * HW + p] = sum * inv_pairs;
    acc += (double)sum;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
  if ((tid & 31) == 0) s_w[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += s_w[w];
    partial[(size_t)v * gridDim.y + blockIdx.y] = t;
  }
}

__global__ void k_w2_fin(const double* __restrict__ partial, int chunks, int n_views, double denom,
                         float* __restrict__ scores) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_views) return;
  double t = 0.0;
  for (int c = 0; c < chunks; ++c) t += partial[(size_t)v * chunks + c];
  scores[v] = (float)(t / denom);
}

}  // namespace
}  // namespace gsr

using namespace gsr;

extern "C" gsr_status gsr_w2_scores(gsr_ctx* ctx, const float* mu, const float* s2, int32_t n_views, int32_t M,
                                    int32_t C, int64_t HW, float* scores, float* map, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!mu || !s2 || !scores) return set_err(ctx, GSR_EINVAL, "gsr_w2_scores: NULL required pointer");
  if (n_views <= 0 || M < 2 || C < 1 || HW < 1)
    return set_err(ctx, GSR_EINVAL, "gsr_w2_scores: need n_views >= 1, M >= 2, C >= 1, HW >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  account(ctx, GSR_STAGE_W2, (M == 5 && C == 4) ? 2 : 1, 8.0 * n_views * (double)M * C * HW + 4.0 * n_views + (map ? 4.0 * n_views * HW : 0));
  StageScope scope(ctx, GSR_STAGE_W2, st);
  if (M == 5 && C == 4) {  // the paper's ensemble (M = 5, 4-channel VAE latents)
    const int chunks = (int)((HW + 1023) / 1024);
    void* part;
    gsr_status s = ensure(ctx, S_SELECT2, (size_t)n_views * chunks * sizeof(double), &part);
    if (s != GSR_OK) return s;
    k_w2_t<5, 4><<<dim3(n_views, chunks), 256, 0, st>>>(mu, s2, HW, (double*)part, map);
    k_w2_fin<<<(n_views + 255) / 256, 256, 0, st>>>((const double*)part, chunks, n_views, (double)HW * 10.0, scores);
  } else {
    k_w2<<<n_views, 512, 0, st>>>(mu, s2, M, C, HW, scores, map);
  }
  return check_cuda(ctx, cudaGetLastError(), "k_w2");
}
