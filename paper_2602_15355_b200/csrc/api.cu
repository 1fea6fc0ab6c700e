// api.cu -- libgsr context, errors, camera builder and the K1 entry point.
#include "gsr_internal.cuh"

#include <cmath>
#include <cstdlib>
#include <cstring>

namespace gsr {

static thread_local std::string g_thread_err;

gsr_status set_err(gsr_ctx* ctx, gsr_status st, const std::string& msg) {
  if (ctx)
    ctx->err = msg;
  else
    g_thread_err = msg;
  return st;
}

gsr_status check_cuda(gsr_ctx* ctx, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return GSR_OK;
  return set_err(ctx, GSR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

gsr_status ensure(gsr_ctx* ctx, Slot s, size_t bytes, void** out) {
  if (bytes == 0) bytes = 256;
  if (ctx->cap[s] < bytes) {
    if (ctx->buf[s]) cudaFree(ctx->buf[s]);  // implicit device sync: no in-flight user
    ctx->buf[s] = nullptr;
    ctx->cap[s] = 0;
    const size_t want = bytes + bytes / 8;  // headroom against small growth steps
    cudaError_t e = cudaMalloc(&ctx->buf[s], want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return set_err(ctx, GSR_ENOMEM, std::string("scratch allocation failed: ") + cudaGetErrorString(e));
    }
    ctx->cap[s] = want;
  }
  *out = ctx->buf[s];
  return GSR_OK;
}

static cudaEvent_t pool_get(gsr_ctx* ctx) {
  if (!ctx->pool.empty()) {
    cudaEvent_t e = ctx->pool.back();
    ctx->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

int stage_begin(gsr_ctx* ctx, int stage, cudaStream_t st) {
  if (!ctx->timing) return -1;
  gsr_ctx::Span s{stage, pool_get(ctx), pool_get(ctx)};
  cudaEventRecord(s.a, st);
  ctx->spans.push_back(s);
  return (int)ctx->spans.size() - 1;
}

void stage_end(gsr_ctx* ctx, int span, cudaStream_t st) {
  if (span < 0 || span >= (int)ctx->spans.size()) return;
  cudaEventRecord(ctx->spans[span].b, st);
}

}  // namespace gsr

using namespace gsr;

extern "C" {

gsr_status gsr_create(gsr_ctx** out, int device) {
  if (!out) return set_err(nullptr, GSR_EINVAL, "gsr_create: NULL out");
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return check_cuda(nullptr, e, "gsr_create: cudaSetDevice");
  gsr_ctx* c = new gsr_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (const char* v = std::getenv("GSR_DKEY64")) c->depth_keys64 = std::atoi(v) != 0;
  if (const char* v = std::getenv("GSR_BWRED")) c->bw_reduce = std::atoi(v);
  if (const char* v = std::getenv("GSR_BWNW")) c->bw_warps = std::atoi(v);
  if (const char* v = std::getenv("GSR_PACK")) c->pack_tile_keys = std::atoi(v);
  if (const char* v = std::getenv("GSR_TSORT"))
    c->tile_sort_mode = std::string(v) == "radix" ? 2 : (std::string(v) == "cs" ? 1 : 0);
  e = cudaMallocHost(&c->host_pinned, 4096);
  if (e != cudaSuccess) {
    delete c;
    return check_cuda(nullptr, e, "gsr_create: cudaMallocHost");
  }
  *out = c;
  return GSR_OK;
}

gsr_status gsr_set_composite_residency(gsr_ctx* ctx, int32_t blocks_per_sm) {
  if (!ctx) return GSR_EINVAL;
  if (blocks_per_sm < 0 || blocks_per_sm > 32)
    return set_err(ctx, GSR_EINVAL, "gsr_set_composite_residency: blocks_per_sm not in [0, 32]");
  ctx->k6_persist = blocks_per_sm;
  return GSR_OK;
}

gsr_status gsr_timing_enable(gsr_ctx* ctx, int enable) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  ctx->timing = enable != 0;
  return GSR_OK;
}

gsr_status gsr_timing_read(gsr_ctx* ctx, double* ms, int64_t* launches, double* bytes) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  double acc[GSR_N_STAGES] = {};
  for (auto& s : ctx->spans) {
    cudaError_t e = cudaEventSynchronize(s.b);
    if (e != cudaSuccess) return check_cuda(ctx, e, "gsr_timing_read");
    float t = 0.f;
    cudaEventElapsedTime(&t, s.a, s.b);
    acc[s.stage] += t;
    ctx->pool.push_back(s.a);
    ctx->pool.push_back(s.b);
  }
  ctx->spans.clear();
  for (int i = 0; i < GSR_N_STAGES; ++i) {
    if (ms) ms[i] = acc[i];
    if (launches) launches[i] = ctx->launches[i];
    if (bytes) bytes[i] = ctx->bytes[i];
    ctx->launches[i] = 0;
    ctx->bytes[i] = 0.0;
  }
  return GSR_OK;
}

gsr_status gsr_destroy(gsr_ctx* ctx) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  cudaSetDevice(ctx->device);
  for (auto& s : ctx->spans) {
    cudaEventDestroy(s.a);
    cudaEventDestroy(s.b);
  }
  for (auto e : ctx->pool) cudaEventDestroy(e);
  for (int s = 0; s < S_NSLOTS; ++s)
    if (ctx->buf[s]) cudaFree(ctx->buf[s]);
  if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
  delete ctx;
  return GSR_OK;
}

gsr_status gsr_upload(gsr_ctx* ctx, void* dst, const void* src, int64_t bytes, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return set_err(ctx, GSR_EINVAL, "gsr_upload: NULL pointer or bytes < 0");
  if (bytes == 0) return GSR_OK;
  return check_cuda(ctx, cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream),
                    "gsr_upload");
}

gsr_status gsr_download(gsr_ctx* ctx, void* dst, const void* src, int64_t bytes, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (bytes < 0 || (bytes > 0 && (!dst || !src)))
    return set_err(ctx, GSR_EINVAL, "gsr_download: NULL pointer or bytes < 0");
  if (bytes == 0) return GSR_OK;
  return check_cuda(ctx, cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream),
                    "gsr_download");
}

const char* gsr_last_error(const gsr_ctx* ctx) { return ctx ? ctx->err.c_str() : g_thread_err.c_str(); }

const char* gsr_version(void) { return "gsr 0.1 sm_100a"; }

int64_t gsr_scratch_bytes(const gsr_ctx* ctx) {
  if (!ctx) return 0;
  int64_t t = 0;
  for (int s = 0; s < S_NSLOTS; ++s) t += (int64_t)ctx->cap[s];
  return t;
}

gsr_status gsr_camera_look_at(double elevation, double azimuth, double radius, const double* target, int32_t width,
                              int32_t height, double focal, double znear, gsr_camera* out) {
  if (!target || !out) return set_err(nullptr, GSR_EINVAL, "gsr_camera_look_at: NULL pointer");
  if (width <= 0 || height <= 0 || !(focal > 0) || !(znear > 0) || !(radius > 0))
    return set_err(nullptr, GSR_EINVAL, "gsr_camera_look_at: non-positive size / focal / znear / radius");
  const double ce = std::cos(elevation), se = std::sin(elevation);
  const double eye[3] = {target[0] + radius * ce * std::cos(azimuth), target[1] + radius * se,
                         target[2] + radius * ce * std::sin(azimuth)};
  double f[3] = {target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]};
  double fl = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
  for (double& x : f) x /= fl;
  double up[3] = {0.0, 1.0, 0.0};
  if (std::fabs(f[1]) > 0.9999) {
    up[1] = 0.0;
    up[2] = 1.0;
  }
  double r[3] = {f[1] * up[2] - f[2] * up[1], f[2] * up[0] - f[0] * up[2], f[0] * up[1] - f[1] * up[0]};
  const double rl = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  for (double& x : r) x /= rl;
  const double d[3] = {f[1] * r[2] - f[2] * r[1], f[2] * r[0] - f[0] * r[2], f[0] * r[1] - f[1] * r[0]};
  const double* rows[3] = {r, d, f};
  for (int i = 0; i < 3; ++i) {
    double ti = 0.0;
    for (int j = 0; j < 3; ++j) {
      out->R[3 * i + j] = (float)rows[i][j];
      ti += rows[i][j] * eye[j];
    }
    out->t[i] = (float)(-ti);
    out->campos[i] = (float)eye[i];
  }
  out->fx = out->fy = (float)focal;
  out->cx = (float)(width / 2.0);
  out->cy = (float)(height / 2.0);
  out->limx = (float)(1.3 * (width / 2.0) / focal);
  out->limy = (float)(1.3 * (height / 2.0) / focal);
  out->znear = (float)znear;
  out->width = width;
  out->height = height;
  return GSR_OK;
}

gsr_status gsr_project(gsr_ctx* ctx, const gsr_gaussians* G, const gsr_camera* cams, int32_t n_views,
                       const gsr_lod* lod, float* render_rec, uint32_t* bin_rec, void* stream) {
  if (!ctx) return GSR_EINVAL;
  DeviceGuard device_guard(ctx);
  if (!G || !cams || !render_rec || !bin_rec) return set_err(ctx, GSR_EINVAL, "gsr_project: NULL required pointer");
  if (G->n < 0 || G->sh_degree < 0 || G->sh_degree > 3)
    return set_err(ctx, GSR_EINVAL, "gsr_project: n < 0 or sh_degree not in [0,3]");
  if (G->n > 0 && (!G->pos_opacity || !G->scale_unc || !G->rot || !G->sh))
    return set_err(ctx, GSR_EINVAL, "gsr_project: NULL Gaussian plane");
  if (n_views <= 0 || n_views > GSR_MAX_VIEWS) return set_err(ctx, GSR_EINVAL, "gsr_project: bad n_views");
  const int W = cams[0].width, H = cams[0].height;
  for (int c = 0; c < n_views; ++c) {
    if (cams[c].width != W || cams[c].height != H || W <= 0 || H <= 0)
      return set_err(ctx, GSR_EINVAL, "gsr_project: mixed or non-positive resolutions in a batch");
    if (!(cams[c].znear > 0.0f)) return set_err(ctx, GSR_EINVAL, "gsr_project: znear <= 0");
  }
  const uint64_t tiles = (uint64_t)((W + kTile - 1) / kTile) * (uint64_t)((H + kTile - 1) / kTile);
  if (tiles * (uint64_t)n_views >= (1ull << 32)) return set_err(ctx, GSR_EINVAL, "gsr_project: V*tiles >= 2^32");
  if (W > 65535 || H > 65535)
    return set_err(ctx, GSR_EINVAL, "gsr_project: W or H > 65535 (16-bit pixel-row fields of the span record)");
  LodParams lp;
  std::memset(&lp, 0, sizeof(lp));
  if (lod) {
    if (lod->levels < 1 || lod->levels > 8 || !(lod->delta > 0.0f) || (G->n > 0 && !lod->tile_level))
      return set_err(ctx, GSR_EINVAL, "gsr_project: bad LOD (levels in [1,8], delta > 0, tile_level required)");
    for (int i = 1; i + 1 < lod->levels; ++i)
      if (!(lod->thresholds[i] > lod->thresholds[i - 1]))
        return set_err(ctx, GSR_EINVAL, "gsr_project: LOD thresholds must increase");
    lp.on = 1;
    lp.levels = lod->levels;
    lp.delta = lod->delta;
    for (int i = 0; i < 7; ++i) lp.D[i] = lod->thresholds[i];
    lp.tile_level = lod->tile_level;
  }
  if (G->n == 0) return GSR_OK;
  CamBatch cb;
  std::memset(&cb, 0, sizeof(cb));
  std::memcpy(cb.c, cams, sizeof(gsr_camera) * (size_t)n_views);
  // algorithmic bytes: parameter planes once per batch + depth / n_tiles planes; the
  // 48-byte render records and 32-byte span records of the visible pairs are added
  // by gsr_bin_sort (it knows N_vis)
  const int planes = 3 + (3 * (G->sh_degree + 1) * (G->sh_degree + 1) + 3) / 4;
  account(ctx, GSR_STAGE_PROJECT, 1, 16.0 * planes * (double)G->n + 8.0 * n_views * (double)G->n);
  StageScope sc(ctx, GSR_STAGE_PROJECT, (cudaStream_t)stream);
  if (lp.on) account(ctx, GSR_STAGE_PROJECT, 0, 16.0 * (double)G->n);
  return check_cuda(ctx, launch_project(*G, cb, lp, n_views, render_rec, bin_rec, (cudaStream_t)stream), "k1_project");
}

}  // extern "C"
