// optim.cu -- NEXT-3 refinement step of UPDATE_GS ("bounded refinement",
// PAPER.md §4.1; Alg. 1): the photometric loss gradient that feeds
// gsr_backward, and the parameter update.
//
//   k_l2    L = (1/N) sum_p sum_ch w_ch (C_p,ch - target_p,ch)^2 over the
//           N = V H W pixels of a batch; dL/dC = (2/N) w (C - target).  One
//           thread per pixel (float4), fixed-order block partials in double.
//   k_adam  Adam (Kingma & Ba 2015, Alg. 1, bias-corrected) per parameter
//           component with a learning rate per (plane, component), then the
//           projection onto the parameters' domain: opacity in [1e-4, 1],
//           scales >= 1e-6, uncertainty >= 0 (DESIGN.md reading: projected
//           Adam on the activated parameters).  HBM-bound: 16 B read + 12 B
//           written per component... (p, g, m, v in; p, m, v out).
#include "gsr_internal.cuh"

#include <cstring>

namespace gsr {
namespace {

constexpr uint32_t FULL = 0xffffffffu;

__global__ void __launch_bounds__(256) k_l2(const float4* __restrict__ img, const float4* __restrict__ tgt,
                                            float4 w, int64_t npx, float scale, float4* __restrict__ dl,
                                            double* __restrict__ partial) {
  __shared__ double s_w[8];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < npx; i += (int64_t)gridDim.x * 256) {
    const float4 a = img[i], b = tgt[i];
    const float dr = a.x - b.x, dg = a.y - b.y, db = a.z - b.z, du = a.w - b.w;
    acc += (double)(w.x * dr * dr) + (double)(w.y * dg * dg) + (double)(w.z * db * db) + (double)(w.w * du * du);
    if (dl) dl[i] = make_float4(2.0f * scale * w.x * dr, 2.0f * scale * w.y * dg, 2.0f * scale * w.z * db,
                                2.0f * scale * w.w * du);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += s_w[k];
    partial[blockIdx.x] = t;
  }
}

__global__ void k_l2_final(const double* __restrict__ partial, int nb, double scale, double* __restrict__ loss) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double t = 0.0;
  for (int b = 0; b < nb; ++b) t += partial[b];
  *loss = t * scale;
}

struct AdamParams {
  float lr[16][4];   // per (plane, component)
  float b1, b2, eps, c1, c2;  // c1 = 1 / (1 - b1^t), c2 = 1 / (1 - b2^t)
};

__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ p, const float4* __restrict__ g,
                                              float4* __restrict__ m, float4* __restrict__ v, int64_t n, int planes,
                                              const __grid_constant__ AdamParams ap) {
  const int64_t total = n * planes;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int pl = (int)(i / n);
    float4 P = p[i], G = g[i], Mv = m[i], Vv = v[i];
    float* pp = &P.x;
    const float* gg = &G.x;
    float* mm = &Mv.x;
    float* vv = &Vv.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      mm[c] = ap.b1 * mm[c] + (1.0f - ap.b1) * gg[c];
      vv[c] = ap.b2 * vv[c] + (1.0f - ap.b2) * gg[c] * gg[c];
      const float mh = mm[c] * ap.c1, vh = vv[c] * ap.c2;
      pp[c] = pp[c] - ap.lr[pl][c] * mh / (sqrtf(vh) + ap.eps);
    }
    if (pl == 0) P.w = fminf(1.0f, fmaxf(1e-4f, P.w));  // opacity
    if (pl == 1) {                                      // scales, uncertainty
      P.x = fmaxf(1e-6f, P.x);
      P.y = fmaxf(1e-6f, P.y);
      P.z = fmaxf(1e-6f, P.z);
      P.w = fmaxf(0.0f, P.w);
    }
    p[i] = P;
    m[i] = Mv;
    v[i] = Vv;
  }
}

}  // namespace
}  // namespace gsr

using namespace gsr;

extern "C" gsr_status gsr_l2_loss(gsr_ctx* ctx, const float* img, const float* target, int64_t n_pixels,
                                  const float* weights, float* dl_dimg, double* loss, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!img || !target || !weights || !loss) return set_err(ctx, GSR_EINVAL, "gsr_l2_loss: NULL required pointer");
  if (n_pixels <= 0) return set_err(ctx, GSR_EINVAL, "gsr_l2_loss: n_pixels <= 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)std::min<int64_t>((n_pixels + 255) / 256, (int64_t)ctx->num_sms * 8);
  void* part;
  gsr_status s;
  if ((s = ensure(ctx, S_OPTIM, (size_t)nb * 8, &part)) != GSR_OK) return s;
  account(ctx, GSR_STAGE_OPTIM, 2, (dl_dimg ? 48.0 : 32.0) * n_pixels);
  StageScope scope(ctx, GSR_STAGE_OPTIM, st);
  const float4 w = make_float4(weights[0], weights[1], weights[2], weights[3]);
  k_l2<<<nb, 256, 0, st>>>((const float4*)img, (const float4*)target, w, n_pixels, (float)(1.0 / (double)n_pixels),
                           (float4*)dl_dimg, (double*)part);
  k_l2_final<<<1, 32, 0, st>>>((const double*)part, nb, 1.0 / (double)n_pixels, loss);
  return check_cuda(ctx, cudaGetLastError(), "k_l2");
}

extern "C" gsr_status gsr_adam_step(gsr_ctx* ctx, float* params, const float* grads, float* m, float* v, int64_t n,
                                    int32_t planes, const float* lr, float beta1, float beta2, float eps,
                                    int32_t step, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!params || !grads || !m || !v || !lr) return set_err(ctx, GSR_EINVAL, "gsr_adam_step: NULL required pointer");
  if (n < 0 || planes < 2 || planes > 16 || step < 1 || !(beta1 >= 0.0f && beta1 < 1.0f) ||
      !(beta2 >= 0.0f && beta2 < 1.0f) || !(eps > 0.0f))
    return set_err(ctx, GSR_EINVAL, "gsr_adam_step: bad n / planes / step / betas / eps");
  if (n == 0) return GSR_OK;
  AdamParams ap;
  std::memset(&ap, 0, sizeof(ap));
  std::memcpy(ap.lr, lr, sizeof(float) * 4 * (size_t)planes);
  ap.b1 = beta1;
  ap.b2 = beta2;
  ap.eps = eps;
  ap.c1 = (float)(1.0 / (1.0 - std::pow((double)beta1, (double)step)));
  ap.c2 = (float)(1.0 / (1.0 - std::pow((double)beta2, (double)step)));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = n * planes;
  account(ctx, GSR_STAGE_OPTIM, 1, 64.0 * total);
  StageScope scope(ctx, GSR_STAGE_OPTIM, st);
  const int nb = (int)std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 16);
  k_adam<<<nb, 256, 0, st>>>((float4*)params, (const float4*)grads, (float4*)m, (float4*)v, n, planes, ap);
  return check_cuda(ctx, cudaGetLastError(), "k_adam");
}
