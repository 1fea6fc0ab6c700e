/*
 * gsr_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * active-view scoring rasterizer (DAV-GSWT, arXiv 2602.15355).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2602_15355_b200/csrc); every constant below is retyped from
 * SURVEY.md Appendix A.
 *
 * What it computes (Alg. 1, §3.5, with the
 * rasterizer readings of SURVEY.md §8(c) -- the paper prints no rasterizer,
 * see DESIGN.md "Readings"):
 *   O1  projection of one Gaussian into one view        orc_project
 *   O4  SH colour (degree <= 3)                         orc_sh_basis / inside orc_project
 *   O2  duplicated (tile|depth, g) keys, emission order  orc_emit_keys
 *   O3  (key, value) lexicographic sort + tile ranges   orc_sort_pairs / orc_ranges
 *   O5  per-pixel front-to-back compositing, tiled      orc_composite_tiled
 *       and brute force over all Gaussians               orc_composite_brute
 *   O6  view score = mean composited uncertainty        (inside the composites)
 *   exp_spec                                             orc_exp_spec
 *   whole view, threaded over views                      orc_render_views
 *
 * Arithmetic: float32, IEEE round-to-nearest, no implicit contraction (built
 * with -ffp-contract=off), fmaf only where §8(c) writes fma(), correctly
 * rounded '/' and sqrtf, expressions evaluated left to right as written in
 * §8(c).  Score sums in double.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  float R[9], t[3], campos[3];
  float fx, fy, cx, cy, limx, limy, znear;
  int32_t width, height;
} orc_camera;

/* NEXT-2 LOD blending parameters (PAPER.md eq:lod_blend L124-127 and its
   clamped form, App. A.4); tile_level [n][4] = (tile centre, level). */
typedef struct {
  int32_t levels;
  float delta;
  float thresholds[7];
  const float* tile_level;
} orc_lod;

/* one projected (view, Gaussian) pair */
typedef struct {
  float u, v, A, B, C, o, unc, r, g, b;
  /* tile-span parameters (O1 step 15): x-shift per row p = b/c,
     conditional x-variance h = det/c, 1/c, and dy of the rightmost point */
  float sp_p, sp_h, sp_ic, sp_dys;
  uint32_t depth_bits, py0, py1, n_tiles; /* py0..py1: pixel rows of the span extent */
} orc_proj;

/* SURVEY.md Appendix A, retyped as literals */
static const float ORC_DILATION = 0.3f;
/* span ellipse q <= ORC_SPAN_T and margin (O1 step 14): 11.1 > 3.33^2 =
   11.0889 > 2 ln 255 = 11.0825, so every pixel with alpha >= 1/255 lies inside
   q <= 11.0889; the 1e-3 relative inflation and the 1/16 px margin absorb the
   float32 rounding of the span arithmetic. */
static const float ORC_SPAN_T = 11.1f;
static const float ORC_SPAN_M = 0.0625f;
static const float ORC_ALPHA_MIN = 1.0f / 255.0f;  /* 0x3b808081 */
static const float ORC_ALPHA_MAX = 0.99f;
static const float ORC_T_STOP = 1e-4f;
static const int ORC_TILE = 16;

static const float SH_C1 = 0.4886025119f;
static const float SH_C2a = 1.0925484306f;
static const float SH_C2b = 0.3153915653f;
static const float SH_C2c = 0.5462742153f;
static const float SH_C3a = 0.5900435899f;
static const float SH_C3b = 2.8906114426f;
static const float SH_C3c = 0.4570457995f;
static const float SH_C3d = 0.3731763326f;
static const float SH_C3e = 1.4453057213f;

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* exp_spec(x), x <= 0 (SURVEY §8(c) O5 note): range reduction by ln2 split
   into hi/lo, degree-7 Taylor polynomial in Horner form, scale by 2^kf. */
float orc_exp_spec(float x) {
  if (x < -80.0f) return 0.0f;
  const float log2e = u2f(0x3fb8aa3bu);
  const float ln2_hi = u2f(0x3f317200u);
  const float ln2_lo = u2f(0x35bfbe8eu);
  float kf = rintf(x * log2e);
  float r = fmaf(kf, -ln2_hi, x);
  r = fmaf(kf, -ln2_lo, r);
  float p = u2f(0x39500d01u);            /* 1/7! */
  p = fmaf(p, r, u2f(0x3ab60b61u));      /* 1/6! */
  p = fmaf(p, r, u2f(0x3c088889u));      /* 1/5! */
  p = fmaf(p, r, u2f(0x3d2aaaabu));      /* 1/4! */
  p = fmaf(p, r, u2f(0x3e2aaaabu));      /* 1/3! */
  p = fmaf(p, r, u2f(0x3f000000u));      /* 1/2! */
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  int k = (int)kf;
  float scale = u2f((uint32_t)(k + 127) << 23);
  return p * scale;
}

/* Real orthonormal SH basis up to degree 3, with Y0 = 1
   (the DC coefficient is the base colour).  dir must be unit length. */
void orc_sh_basis(float x, float y, float z, float Y[16]) {
  float xx = x * x, yy = y * y, zz = z * z;
  float xy = x * y, yz = y * z, xz = x * z;
  Y[0] = 1.0f;
  Y[1] = -SH_C1 * y;
  Y[2] = SH_C1 * z;
  Y[3] = -SH_C1 * x;
  Y[4] = SH_C2a * xy;
  Y[5] = -SH_C2a * yz;
  Y[6] = SH_C2b * (((2.0f * zz) - xx) - yy);
  Y[7] = -SH_C2a * xz;
  Y[8] = SH_C2c * (xx - yy);
  Y[9] = (-SH_C3a * y) * ((3.0f * xx) - yy);
  Y[10] = (SH_C3b * xy) * z;
  Y[11] = (-SH_C3c * y) * (((4.0f * zz) - xx) - yy);
  Y[12] = (SH_C3d * z) * (((2.0f * zz) - (3.0f * xx)) - (3.0f * yy));
  Y[13] = (-SH_C3c * x) * (((4.0f * zz) - xx) - yy);
  Y[14] = (SH_C3e * z) * (xx - yy);
  Y[15] = (-SH_C3a * x) * (xx - (3.0f * yy));
}

/* eq:lod_blend, clamped (App. A.4): a(d, D) = max(0, min(1, 0.5 - (d - D) / (2 delta))).
   Level i fades out around D_i; level i+1 fades in with the complement
   (DESIGN.md reading, "the coarser level taking the complement");
   the weight of a level is the smaller of its fade-in and fade-out. */
float orc_lod_blend(float d, float D, float delta) {
  float a = 0.5f - (d - D) / (2.0f * delta);
  return fminf(1.0f, fmaxf(0.0f, a));
}

float orc_lod_weight(float d, int level, const orc_lod* lod) {
  float w = 1.0f;
  if (level < lod->levels - 1) w = orc_lod_blend(d, lod->thresholds[level], lod->delta);
  if (level > 0) {
    float fin = 1.0f - orc_lod_blend(d, lod->thresholds[level - 1], lod->delta);
    w = fminf(w, fin);
  }
  return w;
}

/* O1 step 15: span [x0, x1) of tile columns of tile row ty.  The pixel rows
   of the tile inside [py0, py1] form the band [ya, yb]; over the band the
   ellipse q <= t, whose x-interval at offset dy is
     p dy -/+ sqrt(h (t - dy^2 / c)),
   reaches furthest right at dy = dys (its rightmost point) and furthest left
   at dy = -dys, so both bounds are taken at those offsets clamped into the
   band.  Columns with a pixel centre in [L, R] (widened by m), clipped to the
   image, give the tile columns.  Empty spans give x0 = x1 = 0. */
void orc_row_span(const orc_proj* p, uint32_t ty, int W, uint32_t* x0, uint32_t* x1) {
  uint32_t ya = ty * 16u > p->py0 ? ty * 16u : p->py0;
  uint32_t yb = ty * 16u + 15u < p->py1 ? ty * 16u + 15u : p->py1;
  float dya = ((float)ya + 0.5f) - p->v;
  float dyb = ((float)yb + 0.5f) - p->v;
  float dr = fminf(fmaxf(p->sp_dys, dya), dyb);
  float dl = fminf(fmaxf(-p->sp_dys, dya), dyb);
  float R = ((p->u + p->sp_p * dr) + sqrtf(fmaxf(0.0f, p->sp_h * (ORC_SPAN_T - (dr * dr) * p->sp_ic)))) + ORC_SPAN_M;
  float L = ((p->u + p->sp_p * dl) - sqrtf(fmaxf(0.0f, p->sp_h * (ORC_SPAN_T - (dl * dl) * p->sp_ic)))) - ORC_SPAN_M;
  float fpx0 = fmaxf(ceilf(L - 0.5f), 0.0f);
  float fpx1 = fminf(floorf(R - 0.5f), (float)(W - 1));
  if (!(fpx0 <= fpx1)) { *x0 = 0; *x1 = 0; return; }
  *x0 = (uint32_t)fpx0 >> 4;
  *x1 = ((uint32_t)fpx1 >> 4) + 1u;
}

/* planes: float32 [P][n][4]; plane 0 (x,y,z,o), 1 (sx,sy,sz,unc), 2 (qw,qx,qy,qz),
   3.. SH slot-major.  Projects Gaussian g into camera cam. */
void orc_project_one(const float* planes, int64_t n, int sh_degree, const orc_camera* cam,
                     const orc_lod* lod, int64_t g, orc_proj* out) {
  memset(out, 0, sizeof(*out));
  const float* po = planes + 4 * g;
  const float* su = planes + 4 * (n + g);
  const float* qq = planes + 4 * (2 * n + g);
  const float mx = po[0], my = po[1], mz = po[2];
  float o = po[3];
  /* NEXT-2: LOD blending scales the opacity by w at camera distance d from the
     Gaussian's tile centre; o w < 1/255 can never reach alpha >= 1/255: cull. */
  if (lod) {
    const float* tl = lod->tile_level + 4 * g;
    int level = (int)tl[3];
    if (level < 0) level = 0;
    if (level > lod->levels - 1) level = lod->levels - 1;
    float ddx = cam->campos[0] - tl[0], ddy = cam->campos[1] - tl[1], ddz = cam->campos[2] - tl[2];
    float d = sqrtf((ddx * ddx + ddy * ddy) + ddz * ddz);
    o = o * orc_lod_weight(d, level, lod);
    if (!(o >= ORC_ALPHA_MIN)) return;
  }
  const float* R = cam->R;
  /* 1. view transform */
  float vx = ((R[0] * mx + R[1] * my) + R[2] * mz) + cam->t[0];
  float vy = ((R[3] * mx + R[4] * my) + R[5] * mz) + cam->t[1];
  float vz = ((R[6] * mx + R[7] * my) + R[8] * mz) + cam->t[2];
  /* 2. near cull */
  if (!(vz > cam->znear)) return;
  /* 3. pixel mean */
  float xn = vx / vz, yn = vy / vz;
  float u = cam->fx * xn + cam->cx;
  float v = cam->fy * yn + cam->cy;
  /* 4. quaternion normalisation */
  float qn = sqrtf(((qq[0] * qq[0] + qq[1] * qq[1]) + qq[2] * qq[2]) + qq[3] * qq[3]);
  float w = qq[0] / qn, x = qq[1] / qn, y = qq[2] / qn, z = qq[3] / qn;
  /* 5. rotation matrix */
  float rm[3][3];
  rm[0][0] = 1.0f - 2.0f * (y * y + z * z);
  rm[0][1] = 2.0f * (x * y - w * z);
  rm[0][2] = 2.0f * (x * z + w * y);
  rm[1][0] = 2.0f * (x * y + w * z);
  rm[1][1] = 1.0f - 2.0f * (x * x + z * z);
  rm[1][2] = 2.0f * (y * z - w * x);
  rm[2][0] = 2.0f * (x * z - w * y);
  rm[2][1] = 2.0f * (y * z + w * x);
  rm[2][2] = 1.0f - 2.0f * (x * x + y * y);
  /* 6. M = R_q S */
  float s[3] = {su[0], su[1], su[2]};
  float M[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M[i][j] = rm[i][j] * s[j];
  /* 7. Sigma = M M^T */
  float S[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) S[i][j] = (M[i][0] * M[j][0] + M[i][1] * M[j][1]) + M[i][2] * M[j][2];
  /* 8. FOV clamp */
  float tx = fminf(cam->limx, fmaxf(-cam->limx, xn)) * vz;
  float ty = fminf(cam->limy, fmaxf(-cam->limy, yn)) * vz;
  /* 9. Jacobian */
  float j00 = cam->fx / vz, j11 = cam->fy / vz, z2 = vz * vz;
  float j02 = -(cam->fx * tx) / z2;
  float j12 = -(cam->fy * ty) / z2;
  /* 10. T = J W (2x3) */
  float T[2][3];
  for (int k = 0; k < 3; ++k) {
    T[0][k] = j00 * R[k] + j02 * R[6 + k];
    T[1][k] = j11 * R[3 + k] + j12 * R[6 + k];
  }
  /* 11. Q = T Sigma */
  float Q[2][3];
  for (int i = 0; i < 2; ++i)
    for (int k = 0; k < 3; ++k) Q[i][k] = (T[i][0] * S[0][k] + T[i][1] * S[1][k]) + T[i][2] * S[2][k];
  /* 12. 2D covariance with dilation */
  float a = ((Q[0][0] * T[0][0] + Q[0][1] * T[0][1]) + Q[0][2] * T[0][2]) + ORC_DILATION;
  float b = (Q[0][0] * T[1][0] + Q[0][1] * T[1][1]) + Q[0][2] * T[1][2];
  float c = ((Q[1][0] * T[1][0] + Q[1][1] * T[1][1]) + Q[1][2] * T[1][2]) + ORC_DILATION;
  /* 13. determinant cull */
  float det = a * c - b * b;
  if (!(det > 0.0f)) return;
  /* 14. span extent: pixel rows whose centre lies within the y-extent of the
     ellipse q <= t (t = ORC_SPAN_T), widened by the margin m */
  const int W = cam->width, H = cam->height;
  float ye = sqrtf(ORC_SPAN_T * c) + ORC_SPAN_M;
  float fpy0 = fmaxf(ceilf((v - ye) - 0.5f), 0.0f);
  float fpy1 = fminf(floorf((v + ye) - 0.5f), (float)(H - 1));
  if (!(fpy0 <= fpy1)) return;
  out->u = u;
  out->v = v;
  out->sp_p = b / c;
  out->sp_h = det / c;
  out->sp_ic = 1.0f / c;
  out->sp_dys = b * sqrtf(ORC_SPAN_T / a);
  out->py0 = (uint32_t)fpy0;
  out->py1 = (uint32_t)fpy1;
  /* 15. tile spans: n_tiles = sum over tile rows of the row's span width */
  uint32_t nt = 0;
  for (uint32_t ty = out->py0 >> 4; ty <= (out->py1 >> 4); ++ty) {
    uint32_t x0, x1;
    orc_row_span(out, ty, W, &x0, &x1);
    nt += x1 - x0;
  }
  if (nt == 0) { memset(out, 0, sizeof(*out)); return; }
  /* 16. conic */
  float inv = 1.0f / det;
  out->A = c * inv;
  out->B = -(b * inv);
  out->C = a * inv;
  out->o = o;
  out->unc = su[3];
  /* 17. depth key */
  out->depth_bits = f2u(vz);
  out->n_tiles = nt;
  /* O4: SH colour */
  float dx = mx - cam->campos[0], dy = my - cam->campos[1], dz = mz - cam->campos[2];
  float len = sqrtf((dx * dx + dy * dy) + dz * dz);
  float Y[16];
  orc_sh_basis(dx / len, dy / len, dz / len, Y);
  int ncoef = (sh_degree + 1) * (sh_degree + 1);
  float rgb[3];
  for (int ch = 0; ch < 3; ++ch) {
    float acc = 0.0f;
    for (int k = 0; k < ncoef; ++k) {
      int flat = 3 * k + ch;
      float coef = planes[4 * ((3 + flat / 4) * n + g) + (flat & 3)];
      acc = (k == 0) ? coef : acc + Y[k] * coef;
    }
    rgb[ch] = fmaxf(0.0f, acc);
  }
  out->r = rgb[0]; out->g = rgb[1]; out->b = rgb[2];
}

void orc_project(const float* planes, int64_t n, int sh_degree, const orc_camera* cam, const orc_lod* lod,
                 orc_proj* out) {
  for (int64_t g = 0; g < n; ++g) orc_project_one(planes, n, sh_degree, cam, lod, g, &out[g]);
}

/* O2: number of keys of one view */
int64_t orc_count_keys(const orc_proj* p, int64_t n) {
  int64_t k = 0;
  for (int64_t g = 0; g < n; ++g) k += p[g].n_tiles;
  return k;
}

/* O2: emit keys of one view (view_in_batch), order g asc, ty asc, tx asc. */
void orc_emit_keys(const orc_proj* p, int64_t n, const orc_camera* cam, int32_t view_in_batch,
                   uint64_t* keys, uint32_t* vals) {
  uint64_t gx = (uint64_t)((cam->width + ORC_TILE - 1) / ORC_TILE);
  uint64_t gy = (uint64_t)((cam->height + ORC_TILE - 1) / ORC_TILE);
  int64_t k = 0;
  for (int64_t g = 0; g < n; ++g) {
    if (p[g].n_tiles == 0) continue;
    for (uint32_t ty = p[g].py0 >> 4; ty <= (p[g].py1 >> 4); ++ty) {
      uint32_t x0, x1;
      orc_row_span(&p[g], ty, cam->width, &x0, &x1);
      for (uint32_t tx = x0; tx < x1; ++tx) {
        uint64_t tile = (uint64_t)view_in_batch * gx * gy + (uint64_t)ty * gx + tx;
        keys[k] = (tile << 32) | (uint64_t)p[g].depth_bits;
        vals[k] = (uint32_t)g;
        ++k;
      }
    }
  }
}

/* NEXT-2b: emit the keys of one view with the Gaussians visited in a given
   order (the cached view-direction ordering) instead of by index: the low
   32 bits of a key are the Gaussian's position in `order`, so the
   (key, value) sort yields every tile's list in that order. */
void orc_emit_keys_order(const orc_proj* p, const uint32_t* order, int64_t len, const orc_camera* cam,
                         int32_t view_in_batch, uint64_t* keys, uint32_t* vals) {
  uint64_t gx = (uint64_t)((cam->width + ORC_TILE - 1) / ORC_TILE);
  uint64_t gy = (uint64_t)((cam->height + ORC_TILE - 1) / ORC_TILE);
  int64_t k = 0;
  for (int64_t i = 0; i < len; ++i) {
    uint32_t g = order[i];
    if (p[g].n_tiles == 0) continue;
    for (uint32_t ty = p[g].py0 >> 4; ty <= (p[g].py1 >> 4); ++ty) {
      uint32_t x0, x1;
      orc_row_span(&p[g], ty, cam->width, &x0, &x1);
      for (uint32_t tx = x0; tx < x1; ++tx) {
        uint64_t tile = (uint64_t)view_in_batch * gx * gy + (uint64_t)ty * gx + tx;
        keys[k] = (tile << 32) | (uint64_t)i;
        vals[k] = g;
        ++k;
      }
    }
  }
}

typedef struct { uint64_t key; uint32_t val; } orc_pair;

static int cmp_pair(const void* a, const void* b) {
  const orc_pair* x = (const orc_pair*)a;
  const orc_pair* y = (const orc_pair*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  if (x->val != y->val) return x->val < y->val ? -1 : 1;
  return 0;
}

/* O3: (key, value) lexicographic sort, in place. */
void orc_sort_pairs(uint64_t* keys, uint32_t* vals, int64_t k) {
  orc_pair* tmp = (orc_pair*)malloc(sizeof(orc_pair) * (size_t)(k > 0 ? k : 1));
  for (int64_t i = 0; i < k; ++i) { tmp[i].key = keys[i]; tmp[i].val = vals[i]; }
  qsort(tmp, (size_t)k, sizeof(orc_pair), cmp_pair);
  for (int64_t i = 0; i < k; ++i) { keys[i] = tmp[i].key; vals[i] = tmp[i].val; }
  free(tmp);
}

/* O3: ranges[t] = [start, end) for t in [0, n_tiles_total); start = number
   of keys whose (view, tile) prefix is smaller than t. */
void orc_ranges(const uint64_t* sorted_keys, int64_t k, int64_t n_tiles_total, uint32_t* ranges /*[T][2]*/) {
  int64_t i = 0;
  for (int64_t t = 0; t < n_tiles_total; ++t) {
    int64_t s = i;
    while (i < k && (int64_t)(sorted_keys[i] >> 32) == t) ++i;
    ranges[2 * t] = (uint32_t)s;
    ranges[2 * t + 1] = (uint32_t)i;
  }
}

/* O5: composite one pixel over an ordered list of Gaussians. */
static void composite_pixel(const orc_proj* p, const uint32_t* order, int64_t len, int px, int py,
                            float out[4], float* t_final, uint32_t* n_contrib, uint64_t* n_eval) {
  float pcx = (float)px + 0.5f, pcy = (float)py + 0.5f;
  float T = 1.0f;
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  uint32_t nc = 0;
  *n_eval = (uint64_t)len; /* entries evaluated: up to and including the stopping one */
  for (int64_t i = 0; i < len; ++i) {
    const orc_proj* q = &p[order[i]];
    float dx = q->u - pcx, dy = q->v - pcy;
    float qf = fmaf(q->A * dx, dx, (q->C * dy) * dy);
    float power = fmaf(-0.5f, qf, -((q->B * dx) * dy));
    if (power > 0.0f) continue;
    float alpha = fminf(ORC_ALPHA_MAX, q->o * orc_exp_spec(power));
    if (alpha < ORC_ALPHA_MIN) continue;
    float tT = T * (1.0f - alpha);
    if (tT < ORC_T_STOP) { *n_eval = (uint64_t)(i + 1); break; }
    float w = alpha * T;
    acc[0] = fmaf(q->r, w, acc[0]);
    acc[1] = fmaf(q->g, w, acc[1]);
    acc[2] = fmaf(q->b, w, acc[2]);
    acc[3] = fmaf(q->unc, w, acc[3]);
    T = tT;
    ++nc;
  }
  out[0] = acc[0]; out[1] = acc[1]; out[2] = acc[2]; out[3] = acc[3];
  *t_final = T;
  *n_contrib = nc;
}

/* O5 + O6, tiled: for each pixel, the sorted values of its tile's range.
   rgbu [H][W][4], t_final / n_contrib [H][W] optional (NULL).  Returns the
   score (double sum of U over all W*H pixels / (W*H)); n_frag[0] = sum n_contrib
   (blended pairs), n_frag[1] = evaluated (pixel, entry) pairs. */
double orc_composite_tiled(const orc_proj* p, const uint32_t* sorted_vals, const uint32_t* ranges_view,
                           const orc_camera* cam, float* rgbu, float* t_final, uint32_t* n_contrib,
                           uint64_t* n_frag) {
  int W = cam->width, H = cam->height;
  int gx = (W + ORC_TILE - 1) / ORC_TILE;
  double sum = 0.0;
  uint64_t frag = 0, ev = 0;
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      int tile = (py / ORC_TILE) * gx + (px / ORC_TILE);
      uint32_t s = ranges_view[2 * tile], e = ranges_view[2 * tile + 1];
      float o4[4], tf; uint32_t nc; uint64_t ne;
      composite_pixel(p, sorted_vals + s, (int64_t)e - (int64_t)s, px, py, o4, &tf, &nc, &ne);
      ev += ne;
      size_t pi = (size_t)py * W + px;
      if (rgbu) memcpy(rgbu + 4 * pi, o4, sizeof(o4));
      if (t_final) t_final[pi] = tf;
      if (n_contrib) n_contrib[pi] = nc;
      sum += (double)o4[3];
      frag += nc;
    }
  if (n_frag) { n_frag[0] = frag; n_frag[1] = ev; }
  return sum / ((double)W * (double)H);
}

/* NEXT-3 support: the blended entries of every pixel of one view, in
   compositing order (the same O5 loop as composite_pixel, recording g
   instead of accumulating).  offsets [H*W+1] (pixel row-major); idx [cap]
   receives the Gaussian indices.  Returns the total count (idx is filled up
   to cap).  The float32 decisions (skip, stop) are exactly the forward's. */
int64_t orc_composite_trace(const orc_proj* p, const uint32_t* sorted_vals, const uint32_t* ranges_view,
                            const orc_camera* cam, int64_t* offsets, uint32_t* idx, int64_t cap) {
  int W = cam->width, H = cam->height;
  int gx = (W + ORC_TILE - 1) / ORC_TILE;
  int64_t k = 0;
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      offsets[(size_t)py * W + px] = k;
      int tile = (py / ORC_TILE) * gx + (px / ORC_TILE);
      uint32_t s = ranges_view[2 * tile], e = ranges_view[2 * tile + 1];
      float pcx = (float)px + 0.5f, pcy = (float)py + 0.5f;
      float T = 1.0f;
      for (uint32_t i = s; i < e; ++i) {
        const orc_proj* q = &p[sorted_vals[i]];
        float dx = q->u - pcx, dy = q->v - pcy;
        float qf = fmaf(q->A * dx, dx, (q->C * dy) * dy);
        float power = fmaf(-0.5f, qf, -((q->B * dx) * dy));
        if (power > 0.0f) continue;
        float alpha = fminf(ORC_ALPHA_MAX, q->o * orc_exp_spec(power));
        if (alpha < ORC_ALPHA_MIN) continue;
        float tT = T * (1.0f - alpha);
        if (tT < ORC_T_STOP) break;
        if (k < cap) idx[k] = sorted_vals[i];
        ++k;
        T = tT;
      }
    }
  offsets[(size_t)W * H] = k;
  return k;
}

/* depth-then-index comparator for the brute-force list */
static const orc_proj* g_brute_p;
static int cmp_depth_index(const void* a, const void* b) {
  uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
  uint32_t di = g_brute_p[i].depth_bits, dj = g_brute_p[j].depth_bits;
  if (di != dj) return di < dj ? -1 : 1;
  return i < j ? -1 : (i > j ? 1 : 0);
}

/* O5 + O6, brute force: every pixel over ALL non-culled Gaussians of the view
   in (depth bits, index) order; no tiles.  Not thread-safe (tiny inputs only). */
double orc_composite_brute(const orc_proj* p, int64_t n, const orc_camera* cam, float* rgbu,
                           float* t_final, uint32_t* n_contrib, uint64_t* n_frag) {
  uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  int64_t len = 0;
  for (int64_t g = 0; g < n; ++g)
    if (p[g].n_tiles > 0) order[len++] = (uint32_t)g;
  g_brute_p = p;
  qsort(order, (size_t)len, sizeof(uint32_t), cmp_depth_index);
  int W = cam->width, H = cam->height;
  double sum = 0.0;
  uint64_t frag = 0, ev = 0;
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      float o4[4], tf; uint32_t nc; uint64_t ne;
      composite_pixel(p, order, len, px, py, o4, &tf, &nc, &ne);
      ev += ne;
      size_t pi = (size_t)py * W + px;
      if (rgbu) memcpy(rgbu + 4 * pi, o4, sizeof(o4));
      if (t_final) t_final[pi] = tf;
      if (n_contrib) n_contrib[pi] = nc;
      sum += (double)o4[3];
      frag += nc;
    }
  free(order);
  if (n_frag) { n_frag[0] = frag; n_frag[1] = ev; }
  return sum / ((double)W * (double)H);
}

/* ---------------------------------------------------------------------------
 * whole-view oracle (O1..O6), one view per thread: used by the bench's
 * cpu_baseline and by parity tests that only need images / scores.
 * ------------------------------------------------------------------------- */
typedef struct {
  const float* planes; int64_t n; int sh_degree;
  const orc_camera* cams; int32_t n_views;
  const orc_lod* lod;   /* opt */
  float* rgbu;          /* opt [V][H][W][4] */
  double* scores;       /* [V] */
  uint64_t* n_frag;     /* [V] */
  int64_t* n_keys;      /* [V] */
  int next; pthread_mutex_t mu;
} orc_job;

static void render_one(orc_job* J, int v) {
  const orc_camera* cam = &J->cams[v];
  int64_t n = J->n;
  orc_proj* p = (orc_proj*)malloc(sizeof(orc_proj) * (size_t)(n > 0 ? n : 1));
  orc_project(J->planes, n, J->sh_degree, cam, J->lod, p);
  int64_t k = orc_count_keys(p, n);
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(k > 0 ? k : 1));
  uint32_t* vals = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(k > 0 ? k : 1));
  orc_emit_keys(p, n, cam, 0, keys, vals);
  orc_sort_pairs(keys, vals, k);
  int gx = (cam->width + ORC_TILE - 1) / ORC_TILE, gy = (cam->height + ORC_TILE - 1) / ORC_TILE;
  uint32_t* ranges = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (size_t)gx * gy);
  orc_ranges(keys, k, (int64_t)gx * gy, ranges);
  size_t img = (size_t)cam->width * cam->height * 4;
  uint64_t nf[2] = {0, 0};
  /* images of one batch share W,H: view v starts at v * img */
  double sc = orc_composite_tiled(p, vals, ranges, cam, J->rgbu ? J->rgbu + (size_t)v * img : NULL,
                                  NULL, NULL, nf);
  J->scores[v] = sc;
  if (J->n_frag) J->n_frag[v] = nf[0];
  if (J->n_keys) J->n_keys[v] = k;
  free(ranges); free(vals); free(keys); free(p);
}

static void* worker(void* arg) {
  orc_job* J = (orc_job*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int v = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (v >= J->n_views) break;
    render_one(J, v);
  }
  return NULL;
}

/* Render and score n_views views (same W,H when rgbu is given) on n_threads
   host threads, one view per thread at a time. */
void orc_render_views(const float* planes, int64_t n, int sh_degree, const orc_camera* cams,
                      int32_t n_views, const orc_lod* lod, int n_threads, float* rgbu, double* scores,
                      uint64_t* n_frag, int64_t* n_keys) {
  orc_job J;
  J.planes = planes; J.n = n; J.sh_degree = sh_degree; J.cams = cams; J.n_views = n_views; J.lod = lod;
  J.rgbu = rgbu; J.scores = scores; J.n_frag = n_frag; J.n_keys = n_keys; J.next = 0;
  pthread_mutex_init(&J.mu, NULL);
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, worker, &J);
  for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&J.mu);
}
