/*
 * gsr.h -- C ABI of libgsr, the B200-native (sm_100a) active-view scoring
 * rasterizer for DAV-GSWT (arXiv 2602.15355).
 *
 * The paper's problem statement (§3.1): candidate camera poses
 * Θ_cand = {θ_j} on a hemisphere, θ = (elevation, azimuth, radius); a scalar
 * uncertainty u(θ) ranks the candidates (§3.2) and the top-k are acquired
 * (Alg. 1).  The north_star (BASELINE.json) makes u(θ) the mean of the
 * per-pixel composited per-Gaussian uncertainty, rendered by tile-based 3DGS
 * forward rasterization (the splat/sort/render pipeline the paper times,
 * PAPER.md L189 and §3.5).  Every numeric rule below is one of the
 * readings listed in DESIGN.md "Readings of the paper".
 *
 * Conventions
 *  - Plain C: no C++ types, no exceptions, no torch types.  Pointers are
 *    DEVICE pointers unless marked [host].  `stream` is a cudaStream_t passed
 *    as void* (NULL = legacy default stream).
 *  - Calls enqueue work on `stream` and return without synchronising unless
 *    marked SYNC.  Outputs are valid once the stream has synchronised.
 *  - Ownership: the caller allocates every input and output; a gsr_ctx owns
 *    only scratch (grown on demand, freed by gsr_destroy).  No pointer is
 *    retained after a call returns.  One context per stream / host thread.
 *  - Errors: every entry point returns a gsr_status; gsr_last_error(ctx)
 *    gives the message of the last non-OK status of that context.  Inputs
 *    must be finite (NaN/Inf is a documented precondition, not checked).
 *    Culled or off-screen Gaussians are not errors (n_tiles = 0).
 */
#ifndef GSR_H
#define GSR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gsr_ctx gsr_ctx;

typedef enum {
  GSR_OK = 0,
  GSR_EINVAL = 1,    /* bad argument: NULL required pointer, n < 0, sh_degree not in [0,3],
                        W/H <= 0, znear <= 0, n_views <= 0 or > GSR_MAX_VIEWS, mixed
                        resolutions in a batch, V*tiles >= 2^32 */
  GSR_ECUDA = 2,     /* a CUDA launch or runtime call failed */
  GSR_ENOMEM = 3,    /* scratch allocation failed */
  GSR_ECAPACITY = 4, /* key capacity too small: *n_keys holds the required size and
                        nothing else was written */
  GSR_EBUDGET = 5    /* k < 1 or k > n - #excluded ("budget error") */
} gsr_status;

/* Largest number of views in one batch (cameras travel as kernel parameters). */
#define GSR_MAX_VIEWS 64
/* Screen tile edge in pixels (BASELINE.json configs[0] "16x16 tiles"). */
#define GSR_TILE 16

/* The Gaussian field 𝒢 ("Gaussian field", per-Gaussian
   uncertainty of the north_star).  Planar float4 planes, each n elements,
   16-byte aligned, device memory:
     pos_opacity [n][4] = (x, y, z, opacity in (0,1])   opacity already activated
     scale_unc   [n][4] = (sx, sy, sz > 0, uncertainty >= 0)   std-devs, activated
     rot         [n][4] = (w, x, y, z)   any non-zero quaternion; normalised in K1
     sh          [P][n][4], P = ceil(3 (d+1)^2 / 4): plane j, element i holds flat
                 coefficients 4j..4j+3 of Gaussian i, flat index = 3*coef + channel;
                 coefficient 0 is the base RGB (DC = colour, no C0 scale/offset). */
typedef struct {
  int64_t n;
  int32_t sh_degree; /* 0..3 */
  int32_t reserved;
  const float* pos_opacity;
  const float* scale_unc;
  const float* rot;
  const float* sh;
} gsr_gaussians;

/* NEXT-2: continuous LOD blending (§3.5 eq:lod_blend L124-127, clamped
   form of App. A.4).  Each Gaussian belongs to one LOD level of one
   tile; at camera distance d = |campos - tile centre| its opacity is scaled by
     w = min(fade_out, fade_in),
     a(d, D)  = min(1, max(0, 0.5 - (d - D) / (2 delta)))      (eq:lod_blend)
     fade_out = a(d, D_level)           (1 for the coarsest level)
     fade_in  = 1 - a(d, D_{level-1})   (1 for level 0)
   i.e. level i fades out around D_i while level i+1 fades in with the
   complement (DESIGN.md reading; SPEC lod-cache S:L563-591).  A Gaussian
   whose scaled opacity o w < 1/255 is culled (it can never reach alpha >=
   1/255).  float32, evaluated in exactly this order on both sides. */
typedef struct {
  int32_t levels;          /* 1..8 */
  float delta;             /* blending bandwidth > 0 */
  float thresholds[7];     /* D_0 < D_1 < ... < D_{levels-2} (world units) */
  const float* tile_level;  /* DEVICE [n][4]: (tile centre x, y, z, level as float) */
} gsr_lod;

/* One pinhole camera, world->camera, OpenCV axes (x right, y down, z forward).
   Built on the host in double and rounded once (gsr_camera_look_at).
   limx = 1.3 (W/2)/fx and limy = 1.3 (H/2)/fy are the EWA FOV clamp. 96 bytes. */
typedef struct {
  float R[9]; /* row-major */
  float t[3];
  float campos[3];
  float fx, fy, cx, cy, limx, limy, znear;
  int32_t width, height;
} gsr_camera;

/* ---- context ------------------------------------------------------------ */
gsr_status gsr_create(gsr_ctx** out, int device);
gsr_status gsr_destroy(gsr_ctx* ctx);
/* Message for the last non-OK status of ctx (ctx may be NULL: thread-global). */
const char* gsr_last_error(const gsr_ctx* ctx);
/* Library version string, e.g. "gsr 0.1 sm_100a". */
const char* gsr_version(void);

/* ---- H1 camera builder (host only) --------------------------------------
   θ = (elevation, azimuth, radius) of PAPER.md L57, looking at `target`
   [host, 3 doubles]:  eye = target + radius (cos e cos a, sin e, cos e sin a);
   f = normalize(target - eye); r = normalize(f x up) with up = +y (or +z if
   |f.y| > 0.9999); d = f x r; R rows (r, d, f); t = -R eye; principal point
   (W/2, H/2); fx = fy = focal.  Computed in double, rounded once.  EINVAL on
   W/H <= 0, focal <= 0, znear <= 0, radius <= 0. */
gsr_status gsr_camera_look_at(double elevation, double azimuth, double radius, const double* target,
                              int32_t width, int32_t height, double focal, double znear,
                              gsr_camera* out /*[host]*/);

/* ---- K1: projection + culling (north_star "projection/culling kernel") ----
   For every (view c, Gaussian g) of the batch: view transform, near cull
   (vz > znear), EWA 2D covariance with 0.3 px^2 dilation and 1.3x FOV clamp,
   det cull, conic, tile spans, SH colour (degree <= 3), depth-key bits
   (O1/O4).  Tile spans (O1 steps 14-15): with Sigma' = [[a,b],[b,c]]
   and t = 11.1 (> 3.33^2 > 2 ln 255), m = 1/16 px, the pixel rows
   py0..py1 are those whose centre lies within v -/+ (sqrt(t c) + m); for each
   tile row ty the band of its pixel rows [ya, yb] gives
     R = ((u + p dr) + sqrt(max(0, h (t - dr^2 / c)))) + m,  dr = clamp(dys, ya+.5-v, yb+.5-v)
     L = ((u + p dl) - sqrt(max(0, h (t - dl^2 / c)))) - m,  dl = clamp(-dys, ...)
   (p = b/c, h = det/c, dys = b sqrt(t/a): the ellipse's x-interval over the
   band), and the span is the tiles holding a pixel column centre in [L, R]
   clipped to the image.  n_tiles = sum of span widths (0 = culled).
   cams        [host] n_views cameras, all with the same W,H (n_views <= GSR_MAX_VIEWS;
               W, H <= 65535)
   lod         OPTIONAL LOD blending (see gsr_lod): opacity o -> o w before every
               other step; EINVAL if levels not in [1,8], delta <= 0, thresholds
               not increasing or tile_level NULL
   render_rec  [V][n][12] float: (u, v, A, B), (C, opacity, uncertainty, tau),
               (r, g, b, ext) -- conic (A,B,C) = inverse 2D covariance; tau =
               -ln(255 opacity) - 1e-3 (alpha-skip pre-test bound); ext = two
               round-up fp16 half-extents of the alpha >= 1/255 ellipse.  Written
               only where n_tiles > 0 (culled records are left untouched).
   bin_rec     uint32 [10 V n], 16-byte aligned:
               words [0, 8Vn): span records [V][n][8] = (u, v, p, h, 1/c, dys,
                               py0 | py1 << 16, n_tiles), written only where n_tiles > 0;
               words [8Vn, 9Vn): depth bits of view-space z [V][n] (0 when culled);
               words [9Vn, 10Vn): n_tiles [V][n] (0 = culled). */
gsr_status gsr_project(gsr_ctx* ctx, const gsr_gaussians* gaussians, const gsr_camera* cams,
                       int32_t n_views, const gsr_lod* lod /* OPTIONAL [host] struct, NULL = off */,
                       float* render_rec, uint32_t* bin_rec, void* stream);

/* ---- K2-K5: tile-count scan, key duplication, radix sort, tile ranges ----
   Produces the (view, tile)-sorted Gaussian lists of the batch.  Key of a
   duplicated entry = ((view_in_batch * gx*gy + ty*gx + tx) << 32) | depth bits,
   value = g; the sorted order is (key, value) lexicographic (O2/O3).
   bin_rec     [10 V n] from gsr_project (same n_views); n = Gaussians per view
   cams        [host] the batch's cameras (same W,H)
   keys        [capacity] uint64, OPTIONAL (NULL: the sorted 64-bit keys are not
               materialised -- the composite needs only vals + ranges)
   vals        [capacity] uint32 sorted values (Gaussian index g)
   capacity    room in keys/vals
   n_keys      [host] SYNC: receives K, the number of duplicated keys; the call
               waits for the count (one 8-byte readback per batch)
   ranges      [V*gx*gy][2] uint32 [start, end) per (view, tile); empty = [s, s)
   keys_unsorted / vals_unsorted  OPTIONAL [capacity]: the duplicated list in
               emission order (view, g ascending, ty ascending, tx ascending over
               each row's span) -- for parity tests
   Returns GSR_ECAPACITY (with *n_keys = K, nothing else written) if K > capacity. */
gsr_status gsr_bin_sort(gsr_ctx* ctx, const uint32_t* bin_rec, int64_t n, const gsr_camera* cams,
                        int32_t n_views, uint64_t* keys, uint32_t* vals, int64_t capacity,
                        int64_t* n_keys, uint32_t* ranges, uint64_t* keys_unsorted,
                        uint32_t* vals_unsorted, void* stream);

/* ---- NEXT-2b: uncertainty-guided cached view-direction orderings ---------
   (§3.5: "multiple view-dependent Gaussian orderings are
   pre-sorted and cached per tile ... tiles with mean uncertainty above a
   threshold tau retain a larger set of cached orderings").  A tile is a
   contiguous index range [tile_start[t], tile_start[t+1]) of the field
   (tile_start [host] int64 [n_tiles + 1], covering [0, n)); bins [host] int32
   [n_tiles] = the tile's number of azimuthal bins (DESIGN.md policy: 16 if
   its mean uncertainty > tau = 0.6, else 8).  Bin k of tile t orders the
   tile's Gaussians by ascending fl32(fl32(x bx) + fl32(z bz)),
   (bx, bz) = float32(cos, sin)(2 pi k / bins[t]), ties by index.
   gsr_order_cache_size: elements of the cache = sum_t bins[t] n_t (host only).
   gsr_build_order_cache: cache [device uint32, that size] = the orderings,
     tile-major then bin-major (global Gaussian indices); once per field.
   gsr_bin_sort_cached: gsr_bin_sort with the per-view depth sort replaced by
     the cached order: per view (host, double) every tile takes the bin
     maximising <h, b_k> (h = the horizontal part of the camera's forward
     direction, ties to the lower k) and the tiles are visited front to back
     by <centre - eye, forward> (centres [host] double [n_tiles][3], ties to
     the lower tile); the visible Gaussians are emitted in that order, so every
     tile list is composited in it (approximate: not the exact depth order).
     Same outputs and errors as gsr_bin_sort (keys: low word = depth bits). */
/* gsr_order_cache_bins: the cache policy of PAPER.md §3.5 L121-122 ("tiles
     whose uncertainty exceeds threshold tau retain a larger set of cached
     orderings"; tau = 0.6, §3.6): bins[t] = hot_bins if the mean
     per-Gaussian uncertainty of tile t (Gaussians [tile_start[t],
     tile_start[t+1]), double sum) exceeds tau, else base_bins.  tile_start
     [host] int64 [n_tiles + 1] covering [0, n); bins [host] int32 [n_tiles].
     SYNC (one n_tiles x 4-byte readback).  EINVAL: NULL pointers, n_tiles not
     in [1, 4096], bins not in [1, 64], ranges not covering [0, n). */
gsr_status gsr_order_cache_bins(gsr_ctx* ctx, const gsr_gaussians* gaussians, const int64_t* tile_start,
                                int32_t n_tiles, float tau, int32_t base_bins, int32_t hot_bins, int32_t* bins,
                                void* stream);
int64_t gsr_order_cache_size(const int64_t* tile_start, int32_t n_tiles, const int32_t* bins);
gsr_status gsr_build_order_cache(gsr_ctx* ctx, const gsr_gaussians* gaussians, const int64_t* tile_start,
                                 int32_t n_tiles, const int32_t* bins, uint32_t* cache, void* stream);
gsr_status gsr_bin_sort_cached(gsr_ctx* ctx, const uint32_t* bin_rec, int64_t n, const gsr_camera* cams,
                               int32_t n_views, const uint32_t* cache, const int64_t* tile_start,
                               int32_t n_tiles, const int32_t* bins, const double* centres, uint64_t* keys,
                               uint32_t* vals, int64_t capacity, int64_t* n_keys, uint32_t* ranges,
                               void* stream);

/* ---- K6: per-pixel front-to-back compositing of RGB + uncertainty ---------
   For pixel (px, py) of view c, over its tile's sorted list: alpha =
   min(0.99, o exp(power)), skip power > 0 or alpha < 1/255, stop before the
   Gaussian that would take T below 1e-4, accumulate w = alpha T into RGB and U
   (O5).  Background 0.
   render_rec, n, vals, ranges: as produced above for the same batch
   rgbu        OPTIONAL [V][H][W][4] float (r, g, b, U)
   t_final     OPTIONAL [V][H][W] float;   n_contrib OPTIONAL [V][H][W] uint32
   gray        OPTIONAL [V][H][W] float: ((r + g) + b) / 3 of the composited pixel,
               the input of gsr_sobel_scores (NEXT-4)
   tile_partial [V][gx*gy] float: sum of U over the tile's in-image pixels
   n_frag      OPTIONAL [2] uint64, ADDED to: [0] blended (pixel, Gaussian) pairs
               ("composited fragments"); [1] (pixel, list entry) pairs the plain
               definition evaluates = sum over pixels of the entries up to and
               including the one that stops it (the whole list if none does) */
gsr_status gsr_composite(gsr_ctx* ctx, const float* render_rec, int64_t n, const uint32_t* vals,
                         const uint32_t* ranges, const gsr_camera* cams, int32_t n_views,
                         float* rgbu, float* t_final, uint32_t* n_contrib, float* gray,
                         float* tile_partial, unsigned long long* n_frag, void* stream);

/* K6 launch shape (performance only; the outputs are identical either way).
   blocks_per_sm = 0 (default): one 64-thread block per 16x4 strip, up to 20
   resident per SM.  blocks_per_sm = k in [1, 32]: a persistent grid of
   k x (SM count) blocks that take strips by an atomic ticket, so the rest of
   each SM stays free for kernels on other streams (the next batch's sorts
   in a multi-stream pipeline: 3,397 vs 3,336 views/s at k = 10 on c3; alone
   on the GPU the same k costs 17 %).  Applies to later
   gsr_composite calls on ctx.  EINVAL: NULL ctx, k outside [0, 32]. */
gsr_status gsr_set_composite_residency(gsr_ctx* ctx, int32_t blocks_per_sm);

/* ---- K7: view score u(θ) = (sum of U over all W*H pixels) / (W*H) ----------
   (north_star "mean composited uncertainty"; the paper's spatial means
   PAPER.md L72 "global average", L78 1/(H_z W_z) sum_p).  Deterministic
   fixed-order reduction of the tile partials (double accumulation).
   scores [V] float. */
gsr_status gsr_score_views(gsr_ctx* ctx, const float* tile_partial, const gsr_camera* cams,
                           int32_t n_views, float* scores, void* stream);

/* ---- K8: next-best-view / top-k (Alg. 1; App. A.2) --
   Order candidates by (score descending, index ascending), drop excluded
   ones, return the first k.  scores [n] float (device, finite);
   exclude [host] OPTIONAL uint8 [n] (non-zero = already captured, never
   returned -- "avoiding redundant sampling"); out_idx [k] int32
   (device).  n <= 16384.  GSR_EBUDGET if k < 1 or k > n - #excluded. */
gsr_status gsr_select_nbv(gsr_ctx* ctx, const float* scores, int32_t n, const uint8_t* exclude,
                          int32_t k, int32_t* out_idx, void* stream);

/* ---- NEXT-4: image-space spatial-frequency term of eq:uncert_img -----------
   (§3.3: "grad is computed using a 3x3 Sobel operator and
   the result is reduced to a scalar via per-pixel Euclidean norm and global
   average"; the image is the rendered view, grayscale = channel mean, with
   replicate padding as SPEC sobel_gradient_scalar S:L241-248 reads it).
   scores[v] = (1/(W H)) sum_p sqrt(Sx(p)^2 + Sy(p)^2) over the gray image.
   gray         [V][H][W] float (gsr_composite's gray output)
   tile_partial [V][gx*gy] float scratch (per-tile sums of magnitudes)
   scores       [V] float.  EINVAL unless W, H >= 3 and 1 <= V <= GSR_MAX_VIEWS.
   The LPIPS term (pretrained AlexNet) is out of scope. */
gsr_status gsr_sobel_scores(gsr_ctx* ctx, const float* gray, const gsr_camera* cams, int32_t n_views,
                            float* tile_partial, float* scores, void* stream);

/* ---- NEXT-3: backward rasterizer (UPDATE_GS, Alg. 1) --------
   Vector-Jacobian product of the batch's composited images: with the
   upstream gradient G = dL/d(r, g, b, U) per pixel, ADDS to `grads` the
   gradient of L = sum_v sum_p <G_v(p), C_v(p)> w.r.t. every Gaussian
   parameter, in the field's plane layout:
     plane 0 (d mean xyz, d opacity), plane 1 (d scale xyz, d uncertainty),
     plane 2 (d raw quaternion wxyz, through the normalisation), planes 3..
     (d SH coefficients, flat index 3*coef + channel).
   The blended (pixel, Gaussian) pairs and their order are the forward's (same
   float32 decisions); the image is differentiated between those decisions
   (alpha clamp, FOV clamp and max(0, colour) pass gradient only where
   inactive).  Inputs are the forward products of THIS batch: render_rec /
   bin_rec (gsr_project, same lod), vals / ranges (gsr_bin_sort), rgbu (the
   forward image, gsr_composite), dl_drgbu [V][H][W][4].  Float atomics: the
   sums are not bit-deterministic.  grads [P][n][4] float (device). */
gsr_status gsr_backward(gsr_ctx* ctx, const gsr_gaussians* gaussians, const gsr_camera* cams, int32_t n_views,
                        const gsr_lod* lod, const float* render_rec, const uint32_t* bin_rec,
                        const uint32_t* vals, const uint32_t* ranges, const float* rgbu,
                        const float* dl_drgbu, float* grads, void* stream);

/* ---- NEXT-3: refinement step of UPDATE_GS ("bounded refinement (5k
   iterations per inserted image)", §4.1) ----------------------
   gsr_l2_loss: L = (1/N) sum_p sum_ch w_ch (img - target)^2 over N = n_pixels
     (r, g, b, U) pixels; dl_dimg OPTIONAL receives dL/dimg = (2/N) w (img -
     target) (the upstream gradient of gsr_backward); loss [device, 1 double].
     weights [host] 4 floats.
   gsr_adam_step: Adam (Kingma & Ba 2015, bias-corrected, step >= 1) on the
     field planes params [planes][n][4] with grads, moments m, v of the same
     layout, a learning rate per (plane, component) lr [host] [planes][4];
     afterwards opacity is clamped to [1e-4, 1], scales to >= 1e-6 and the
     uncertainty to >= 0 (projection onto the activated parameters' domain).
   Pruning and densification are out of scope. */
gsr_status gsr_l2_loss(gsr_ctx* ctx, const float* img, const float* target, int64_t n_pixels, const float* weights,
                       float* dl_dimg, double* loss, void* stream);
gsr_status gsr_adam_step(gsr_ctx* ctx, float* params, const float* grads, float* m, float* v, int64_t n,
                         int32_t planes, const float* lr, float beta1, float beta2, float eps, int32_t step,
                         void* stream);

/* ---- NEXT-1: latent-space ensemble disagreement (PAPER.md eq:w2_pixel,
   §3.3) ---------------------------------------------------------------
   For each candidate view v: W2 = (1/(H_z W_z)) sum_p (1/C(M,2)) sum_{i<j}
   ( ||mu_{i,p} - mu_{j,p}||^2 + sum_c (s2_{i,p,c} + s2_{j,p,c} - 2 sqrt(s2_{i,p,c} s2_{j,p,c})) ),
   each sample m a diagonal-Gaussian latent (mean mu, per-channel variance s2).
   mu, s2   [V][M][C][HW] float (device), s2 >= 0
   scores   [V] float;  map OPTIONAL [V][HW] float per-location divergence
   EINVAL unless V >= 1, M >= 2, C >= 1, HW >= 1.  The LPIPS term of
   eq:uncert_latent is not part of this call (no pretrained network). */
gsr_status gsr_w2_scores(gsr_ctx* ctx, const float* mu, const float* s2, int32_t n_views, int32_t M, int32_t C,
                         int64_t HW, float* scores, float* map, void* stream);

/* ---- utility: the onesweep LSD radix sort used by gsr_bin_sort ------------
   Stable sort of (key, value) pairs by key bits [begin_bit, end_bit), 8-bit
   digits, one upfront histogram pass + one decoupled-lookback scatter pass
   per digit.  Keys/vals in are not modified; out buffers receive the result.
   0 <= begin_bit < end_bit <= 64; n < 2^31.  Exposed for standalone tests and
   the sort roofline measurement. */
gsr_status gsr_sort_pairs_u64(gsr_ctx* ctx, const uint64_t* keys_in, const uint32_t* vals_in,
                              uint64_t* keys_out, uint32_t* vals_out, int64_t n, int32_t begin_bit,
                              int32_t end_bit, void* stream);

/* ---- host staging (the end-to-end path: inputs in from host memory, the
   result back out, on the pipeline's own stream) ---------------------------
   gsr_upload:   bytes from HOST src to DEVICE dst, enqueued on `stream`.
   gsr_download: bytes from DEVICE src to HOST dst, enqueued on `stream`.
   Asynchronous when the host buffer is page-locked (cudaHostAlloc /
   cudaHostRegister); with pageable memory the copy returns only once the
   host buffer may be reused (cudaMemcpyAsync semantics).  The caller owns
   both buffers and keeps them alive until the stream has synchronised.
   bytes == 0 is a no-op.  EINVAL: NULL ctx / pointer with bytes > 0,
   bytes < 0; ECUDA: the copy failed (e.g. dst / src in the wrong space). */
gsr_status gsr_upload(gsr_ctx* ctx, void* dst, const void* src /*[host]*/, int64_t bytes, void* stream);
gsr_status gsr_download(gsr_ctx* ctx, void* dst /*[host]*/, const void* src, int64_t bytes, void* stream);

/* ---- utility: bytes of scratch the context currently holds (diagnostics) */
int64_t gsr_scratch_bytes(const gsr_ctx* ctx);

/* ---- diagnostics: per-stage kernel launch counts, CUDA-event timing and
   algorithmic HBM bytes.  Stages: */
enum {
  GSR_STAGE_PROJECT = 0,    /* K1 */
  GSR_STAGE_COMPACT = 1,    /* K2 tile-count scan + visible compaction */
  GSR_STAGE_DEPTH_SORT = 2, /* K4a onesweep passes over (view, depth) keys */
  GSR_STAGE_EMIT = 3,       /* K3 key duplication + warp-aggregated tile counts */
  GSR_STAGE_RANGES = 4,     /* K5 tile ranges + tile-sort histograms */
  GSR_STAGE_TILE_SORT = 5,  /* K4b onesweep passes over (view, tile) keys */
  GSR_STAGE_COMPOSITE = 6,  /* K6 */
  GSR_STAGE_SCORE = 7,      /* K7 */
  GSR_STAGE_SELECT = 8,     /* K8 */
  GSR_STAGE_SORT_U64 = 9,   /* utility sort (histogram + passes) */
  GSR_STAGE_W2 = 10,        /* NEXT-1 latent W2 scorer */
  GSR_STAGE_SOBEL = 11,     /* NEXT-4 Sobel image term */
  GSR_STAGE_BACKWARD = 12,  /* NEXT-3 backward rasterizer K6b (+ the grad2d clear) */
  GSR_STAGE_OPTIM = 13,     /* NEXT-3 loss gradient + Adam step */
  GSR_STAGE_BACKWARD_PROJECT = 14, /* NEXT-3 K1b: chain rule to the field parameters */
  GSR_N_STAGES = 15
};
/* enable != 0: bracket every stage with CUDA events on its launch stream. */
gsr_status gsr_timing_enable(gsr_ctx* ctx, int enable);
/* SYNC.  For each stage since the last read: device milliseconds (sum of the
   event-bracketed spans; 0 when timing is off), kernel launches, algorithmic
   HBM bytes (the bytes the step must move).
   Any output pointer may be NULL.  Resets the accumulators. [host] arrays of
   GSR_N_STAGES. */
gsr_status gsr_timing_read(gsr_ctx* ctx, double* ms, int64_t* launches, double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* GSR_H */
