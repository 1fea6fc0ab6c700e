// select.cu -- K8: next-best-view / top-k selection (O7;
// PAPER.md Alg. 1 "top-k poses by u(θ)", App. A.2).
//
// One block bitonic-sorts 64-bit composite keys
//   (~orderable(score) << 32) | index      (excluded -> UINT64_MAX)
// ascending, i.e. score descending then index ascending, and writes the first
// k indices.  N_θ <= 16384 fits one block's shared memory.
#include "gsr_internal.cuh"

namespace gsr {
namespace {

__global__ void __launch_bounds__(1024) k8_select(const float* __restrict__ scores, int n, int P,
                                                  const uint8_t* __restrict__ exclude, int k,
                                                  int32_t* __restrict__ out) {
  extern __shared__ unsigned long long s_key[];
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    unsigned long long key = ~0ull;
    if (i < n && !(exclude && exclude[i])) {
      const uint32_t b = __float_as_uint(scores[i] + 0.0f);  // -0 -> +0
      const uint32_t ob = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
      key = ((unsigned long long)(~ob) << 32) | (uint32_t)i;
    }
    s_key[i] = key;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const unsigned long long a = s_key[i], b = s_key[j];
          if ((a > b) == up) {
            s_key[i] = b;
            s_key[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = (int32_t)(uint32_t)(s_key[i] & 0xffffffffu);
}

}  // namespace
}  // namespace gsr

using namespace gsr;

extern "C" gsr_status gsr_select_nbv(gsr_ctx* ctx, const float* scores, int32_t n, const uint8_t* exclude, int32_t k,
                                     int32_t* out_idx, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!scores || !out_idx) return set_err(ctx, GSR_EINVAL, "gsr_select_nbv: NULL required pointer");
  if (n <= 0 || n > 16384) return set_err(ctx, GSR_EINVAL, "gsr_select_nbv: n must be in [1, 16384]");
  int excluded = 0;
  if (exclude)
    for (int i = 0; i < n; ++i) excluded += exclude[i] != 0;
  if (k < 1 || k > n - excluded) return set_err(ctx, GSR_EBUDGET, "gsr_select_nbv: k < 1 or k > n - #excluded");
  cudaStream_t st = (cudaStream_t)stream;
  void* dex = nullptr;
  gsr_status s;
  if (exclude) {
    if ((s = ensure(ctx, S_SELECT, (size_t)n, &dex)) != GSR_OK) return s;
    if ((s = check_cuda(ctx, cudaMemcpyAsync(dex, exclude, (size_t)n, cudaMemcpyHostToDevice, st), "exclude H2D")) !=
        GSR_OK)
      return s;
  }
  int P = 1;
  while (P < n) P <<= 1;
  const size_t smem = (size_t)P * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k8_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if ((s = check_cuda(ctx, e, "k8 smem attribute")) != GSR_OK) return s;
  }
  account(ctx, GSR_STAGE_SELECT, 1, 4.0 * n + 4.0 * k);
  StageScope scope(ctx, GSR_STAGE_SELECT, st);
  k8_select<<<1, 1024, smem, st>>>(scores, n, P, (const uint8_t*)dex, k, out_idx);
  return check_cuda(ctx, cudaGetLastError(), "k8_select");
}
