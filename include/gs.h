/*
 * gs.h — C-ABI of the B200-native differentiable Gaussian-splatting rasterizer
 * (the hot path of Gaussian-SLAM, arXiv 2312.10070).
 *
 * Citation shorthand: "P:n" = PAPER.md line n (the paper's LaTeX), "S:n" =
 * SPEC.md line n, "SURVEY §x" = /root/repo/SURVEY.md.  Readings of silent or
 * ambiguous passages ("R1".."R26") are listed in DESIGN.md §3.
 *
 * Conventions shared by every entry point
 * ----------------------------------------
 *  - Every pointer is a DEVICE pointer to caller-owned memory unless marked
 *    (host).  The library never allocates, frees or synchronises inside a hot
 *    call; every call is asynchronous on `stream` (a cudaStream_t passed as
 *    void*, NULL = legacy default stream).
 *  - All float arrays are IEEE fp32, all "[n][4]" arrays are 16-byte aligned
 *    float4 records (misalignment is GS_ERR_INVALID_ARG).
 *  - Images are planar, row-major: color[3][H][W], depth[H][W], ...; pixel
 *    (i, j) = (column, row) is sampled at the point (i, j) (R3).
 *  - Tiles are 16x16 pixels, TX = ceil(W/16), TY = ceil(H/16), tile id =
 *    ty*TX + tx; edge tiles are partial (R9).
 *  - Return value: GS_OK or a negative GS_ERR_* code.  Host-side validation
 *    failures never touch the device.  GS_ERR_CUDA carries the CUDA error
 *    string in gs_last_error() (thread-local).  Device-side conditions
 *    (non-finite projection, pair-capacity overflow) do not fail the call:
 *    they increment gs_counters, which the caller reads asynchronously.
 *  - Thread-safe across streams: there is no global mutable state.
 */
#ifndef GS_H
#define GS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ABI_VERSION 2

/* Rasterizer constants (fp32 bit patterns in DESIGN.md R11). */
#define GS_TILE 16                   /* 16x16 pixel tiles           */
#define GS_DILATION 0.3f             /* +0.3 px^2 low-pass dilation (R7)    */
#define GS_ALPHA_MAX 0.999f          /* alpha clamp (R11)                   */
#define GS_ALPHA_MIN (1.0f / 255.0f) /* skip alpha < 1/255 (R11)            */
#define GS_T_EPS 1e-4f               /* stop after T < 1e-4 (R11)           */

/* Status codes. */
#define GS_OK 0
#define GS_ERR_INVALID_ARG (-1)
#define GS_ERR_WORKSPACE (-2)
#define GS_ERR_CUDA (-3)
#define GS_ERR_UNSUPPORTED (-4)

/* gs_render_bwd flags. */
#define GS_GRAD_PARAMS 1u /* per-Gaussian parameter gradients (mapping) */
#define GS_GRAD_POSE 2u   /* camera-pose partials (tracking)           */
#define GS_BWD_PIXELS_ONLY 4u /* run only the per-pixel phase (S5)                 */
#define GS_BWD_GAUSS_ONLY 8u  /* run only the per-Gaussian phase (S6)              */
#define GS_BWD_ATOMIC_ACC 16u /* S6 adds into g_* with atomic vector adds:  calls on
                                 several streams may accumulate into the same arrays
                                 concurrently (summation order unspecified)        */

/* Pinhole camera, passed by value (R4, R5). */
typedef struct gs_camera {
  int32_t width, height; /* pixels, > 0                                  */
  float fx, fy;          /* focal lengths in pixels, > 0                 */
  float cx, cy;          /* principal point in pixels                    */
  float z_near, z_far;   /* keep a Gaussian iff z_near <= p_z <= z_far   */
} gs_camera;

/* World->camera rigid transform T_wc: p = R mu + t, R row-major.
 * Always passed as a DEVICE pointer so the tracking loop can update it in
 * place (gs_pose_grad). 48 bytes. */
typedef struct gs_view {
  float R[9];
  float t[3];
} gs_view;

/* Gaussian parameters (R18, R19), SoA of
 * float4 records, all [n][4]:
 *   mean_opa = (mu_x, mu_y, mu_z, opacity logit)   o = sigmoid(logit)
 *   quat     = (w, x, y, z)                        normalised inside gs_project
 *   logscale = (ln s_x, ln s_y, ln s_z, unused)    s = exp(logscale)
 *   rgb      = (r, g, b, unused)                   raw RGB, no activation   */
typedef struct gs_params {
  const float *mean_opa;
  const float *quat;
  const float *logscale;
  const float *rgb;
  int32_t n; /* >= 0 */
} gs_params;

/* Per-Gaussian projection results written by gs_project (Eqs. 1-2,
 * P:123-131), all indexed by Gaussian id:
 *   uv            [n][2] fp64  splatted mean mu^I = (u, v) in pixels (R1, H2)
 *   conic_o       [n][4] fp32  (A, B, C, o): (Sigma^I + 0.3 I)^-1 = [[A,B],[B,C]]
 *   coef          [n][4] fp32  (a', b', d', log2 o) with
 *                              sigma*log2(e) = (a' dx + b' dy)^2 + (d' dy)^2
 *   rgbz          [n][4] fp32  (r, g, b, p_z) — colour and camera depth (R12)
 *   depth         [n]    fp32  RN(p_z), the sort key; +inf when culled
 *   rect          [n][4] int16 inclusive tile rect (x0, y0, x1, y1);
 *                              (0, 0, -1, -1) when culled
 *   tiles_touched [n]    int32 (x1-x0+1)(y1-y0+1), 0 when culled
 * Fields of culled Gaussians other than depth/rect/tiles_touched are
 * unspecified. */
typedef struct gs_proj {
  double *uv;
  float *conic_o;
  float *coef;
  float *rgbz;
  float *depth;
  int16_t *rect;
  int32_t *tiles_touched;
} gs_proj;

/* Device-side diagnostic counters, accumulated (never reset by the library). */
typedef struct gs_counters {
  int64_t n_nonfinite; /* non-finite or singular projections, culled */
  int64_t n_culled;    /* all culled Gaussians (near/far, off-screen, non-finite)    */
  int64_t n_overflow;  /* gs_bin_sort calls whose pair count exceeded capacity      */
  int64_t reserved;
} gs_counters;

/* Adam step on the left-perturbation twist of T_wc (host, by pointer).
 * Defaults: lr_trans 2e-3 m, lr_rot 1e-3 rad, 0.9, 0.999, 1e-8.
 * beta1, beta2, eps are fp64 (as in gs_adam_cfg): 1 - beta is formed without
 * the fp32 rounding of 0.999 (1 - fp32(0.999) = 1.0000467e-3). */
typedef struct gs_pose_step {
  float lr_trans, lr_rot;
  double beta1, beta2, eps;
} gs_pose_step;

/* ---------------------------------------------------------------------- */
/* Library / device queries (host).                                        */

/* ABI version (GS_ABI_VERSION). */
int gs_version(void);

/* Last error message of the calling thread; never NULL. */
const char *gs_last_error(void);

/* Returns GS_OK iff `device` is an sm_100 (B200-class) GPU; writes its SM
 * count to *sm_count (host, nullable). GS_ERR_UNSUPPORTED otherwise. */
int gs_check_device(int device, int *sm_count);

/* Number of tiles of a camera: ceil(W/16)*ceil(H/16); 0 on invalid camera. */
int32_t gs_num_tiles(gs_camera cam);

/* Workspace bytes gs_bin_sort needs for n Gaussians, a pair capacity and
 * camera `cam`: ~12 bytes per pair of capacity (scratch of the exact sort of
 * long tile lists) + 12 bytes per tile.  0 if unsupported (> 2^21 tiles or
 * capacity >= 2^31 - 1). */
size_t gs_binsort_workspace_bytes(int32_t n, int64_t capacity, gs_camera cam);

/* Workspace bytes gs_loss needs for camera `cam`. */
size_t gs_loss_workspace_bytes(gs_camera cam);

/* Workspace bytes gs_render_bwd needs for n Gaussians: the grad2d scratch
 * [n][12] fp32 = (u, v, A, B), (C, p_z, logit, 0), (r, g, b, 0) per Gaussian.
 * The caller zeroes it ONCE before first use; the per-Gaussian phase zeroes
 * every record it consumes, so it is zero again when gs_render_bwd returns
 * (no memset per call). */
size_t gs_bwd_workspace_bytes(int32_t n);

/* Number of pose-partial records [count][12] gs_render_bwd writes with
 * GS_GRAD_POSE for n Gaussians. */
int32_t gs_pose_partials_count(int32_t n);

/* ---------------------------------------------------------------------- */
/* S1 — EWA projection (Eqs. 1-2).
 *
 * Per Gaussian: q^ = q/|q|, R_q(q^), s = exp(logscale), Sigma = R_q S^2 R_q^T;
 * p = R mu + t; culled iff not z_near <= p_z <= z_far; u = fx p_x/p_z + cx,
 * v = fy p_y/p_z + cy; Sigma^I = J R Sigma R^T J^T + 0.3 I with the unclamped
 * perspective Jacobian J (R6); conic = (Sigma^I)^-1 (culled if det <= 0);
 * o = sigmoid(logit); tile rect = tiles meeting the box of the region where
 * alpha~ = o exp(-sigma) >= 1/255 (half-widths sqrt(2 tau a), sqrt(2 tau c),
 * tau = ln(o / (1/255)), R8'), clamped to the image (culled if empty or
 * tau <= 0).  The decision path (p, u, v, Sigma^I, tau, rect) is evaluated in
 * IEEE fp64 in the operation order of
 * DESIGN.md §3 R1 without FMA contraction, so tile and sort indices are
 * reproducible bit-for-bit.
 *   p      (device) parameters, n >= 0
 *   view   (device) T_wc
 *   cam    camera by value
 *   out    (device) output arrays, each sized for p.n
 *   cnt    (device) counters, nullable
 * Errors: GS_ERR_INVALID_ARG on null arrays (n > 0), bad camera, misalignment. */
int gs_project(gs_params p, const gs_view *view, gs_camera cam, gs_proj out,
               gs_counters *cnt, void *stream);

/* S2 — tile binning and depth ordering ("m ordered Gaussians"; S:132,
 * S:142; R10).
 *
 * Emits one (tile, Gaussian) pair per tile of each visible Gaussian's rect and
 * orders all pairs by the key (tile asc, fp32 depth asc, Gaussian id asc):
 * pairs are emitted into per-tile segments, then every segment is sorted
 * exactly on (depth bits, id) (bit-deterministic whatever the order of the
 * emission's atomics).
 *   pr.depth, pr.rect, pr.tiles_touched (device) inputs from gs_project
 *   ws/ws_bytes   (device) workspace >= gs_binsort_workspace_bytes(n, capacity, cam)
 *   capacity      length of sorted_idx
 *   sorted_idx    (device) [capacity] Gaussian ids, tile-major
 *   tile_range    (device) [T][2] int32 [start, end) into sorted_idx
 *   tile_order    (device, nullable) [T] int32 tile ids by descending list
 *                 length (64 buckets; order within a bucket unspecified): a
 *                 scheduling hint for gs_render_fwd / gs_render_bwd, which
 *                 then start the heaviest tiles first (no effect on results);
 *                 NULL (a caller that reuses an earlier work order) also
 *                 takes the cheaper multi-CTA counts step
 *   n_pairs       (device) [1] int64 total pair count P
 *   cnt           (device) counters, nullable
 * If P > capacity, n_overflow is incremented, every tile range is set empty
 * and sorted_idx is left untouched (the caller re-sizes and repeats). */
int gs_bin_sort(gs_proj pr, int32_t n, gs_camera cam, void *ws, size_t ws_bytes,
                int64_t capacity, int32_t *sorted_idx, int32_t *tile_range,
                int32_t *tile_order, int64_t *n_pairs, gs_counters *cnt, void *stream);

/* S3 — front-to-back alpha compositing (Eqs. 3, 4, 6; P:133-141, P:161-166;
 * S:129-138; R11-R15).
 *
 * Per pixel over its tile's ordered list: Delta = (u - i, v - j);
 * alpha = min(o exp(-1/2 Delta^T conic Delta), 0.999); skip if alpha < 1/255;
 * C += c alpha T; D += p_z alpha T; A += alpha T; T <- T - alpha T (one
 * fused rounding); stop after compositing an entry that leaves T < 1e-4.
 * Background is zero.
 *   tile_order (device, nullable) from gs_bin_sort: launch order of the tiles
 *   color     (device) [3][H][W]    depth, alpha, T_final (device) [H][W]
 *   n_contrib (device) [H][W] int32 (position in the tile list of the last
 *             composited entry) + 1, 0 if none
 *   stats     (device, nullable) [2][H][W] int32: entries scanned, entries
 *             composited — the per-pixel counts of SURVEY §8(d)
 *   tile_work (device, nullable) [T] int32: the backward's work proxy per
 *             tile for gs_tile_order: the largest n_contrib of the tile
 *             (the backward's warps walk back from their strip's largest). */
int gs_render_fwd(gs_proj pr, const int32_t *sorted_idx, const int32_t *tile_range,
                  const int32_t *tile_order, gs_camera cam, float *color, float *depth,
                  float *alpha, float *T_final, int32_t *n_contrib, int32_t *stats,
                  int32_t *tile_work, void *stream);

/* S3 with S4's gradient fused (tracking, BJ.configs[2]; SURVEY S4 "fusable"):
 * gs_render_fwd, then in the same kernel, per pixel, the gradient maps of
 * gs_loss with weight 1:  dL_dcolor = scales[0] sign(C^ - C*),
 * dL_ddepth = scales[1] sign(D^ - D*) where D* > 0, else 0 (sign(0) = 0) —
 * the same fp32 values gs_loss writes.  The loss VALUE is not computed (the
 * tracking update needs only the gradient).  Arguments as gs_render_fwd
 * (no stats) plus:
 *   tgt_color [3][H][W], tgt_depth [H][W] (device) the frame's targets
 *   scales    (device) [4] from gs_loss_scales for this target frame
 *   dL_dcolor [3][H][W], dL_ddepth [H][W] (device) written
 *   loss_part (device, nullable) [T][2] fp64: per tile, sum |C^ - C*| over
 *             its pixels and channels, sum |D^ - D*| over its valid pixels
 *             (fixed order); gs_loss_from_tiles turns them into the loss.
 *   tile_done (device, nullable) [T + 1] uint32, zero on first use:
 *             per-tile completion flags [0, T) for the NEXT call on the
 *             stream being a gs_render_bwd with the same tile_done (it then
 *             starts while this forward finishes, each tile after its own
 *             forward tile, and re-arms the flags), and at [T] the count of
 *             capped waits that timed out (see gs_render_bwd; 0 unless the
 *             contract below is broken).  Every call given tile_done must be
 *             followed by exactly one such backward. */
int gs_render_fwd_l1(gs_proj pr, const int32_t *sorted_idx, const int32_t *tile_range,
                     const int32_t *tile_order, gs_camera cam, float *color, float *depth,
                     float *alpha, float *T_final, int32_t *n_contrib, int32_t *tile_work,
                     const float *tgt_color, const float *tgt_depth, const float *scales,
                     float *dL_dcolor, float *dL_ddepth, double *loss_part, uint32_t *tile_done,
                     void *stream);

/* Scheduling utility: tile ids by descending work (64 buckets of max/64, order
 * inside a bucket unspecified), e.g. from gs_render_fwd's tile_work for
 * gs_render_bwd.  work (device) [T] >= 0; order (device) [T]. */
int gs_tile_order(const int32_t *work, int32_t T, int32_t *order, void *stream);

/* S4 — L1 colour + L1 depth loss (Eqs. 9, 10 L1 part, 12; P:178-202;
 * S:256-264; R20, R21).
 *
 * L_c = sum w |C^ - C*| / (3HW);  L_d = sum_{D* > 0} w |D^ - D*| / |V|;
 * loss = (lambda_color L_c + lambda_depth L_d, L_c, L_d).
 * dL_dcolor = lambda_color w sign(C^ - C*) / (3HW);
 * dL_ddepth = lambda_depth w sign(D^ - D*) / |V| on valid pixels, 0 else;
 * sign(0) = 0; |V| = 0 gives L_d = 0 and a zero depth gradient.
 *   weight (device, nullable) [H][W] per-pixel weight w (1 when NULL)
 *   ws     (device) >= gs_loss_workspace_bytes(cam)
 *   loss   (device) [3]
 * The loss value is bit-deterministic (fixed-order two-stage reduction). */
int gs_loss(gs_camera cam, const float *color, const float *depth,
            const float *tgt_color, const float *tgt_depth, const float *weight,
            float lambda_color, float lambda_depth, void *ws, size_t ws_bytes,
            float *loss, float *dL_dcolor, float *dL_ddepth, void *stream);

/* The two gradient scales of gs_loss for a target frame (weight 1):
 * scales[0] = lambda_color / (3HW), scales[1] = lambda_depth / |V| (0 if
 * |V| = 0), scales[2] = |V| = #{D* > 0} (exact in fp32: HW < 2^24),
 * scales[3] = 0; computed once per frame for gs_render_fwd_l1.
 *   ws (device) >= gs_loss_workspace_bytes(cam); scales (device) [4]. */
int gs_loss_scales(gs_camera cam, const float *tgt_depth, float lambda_color, float lambda_depth,
                   void *ws, size_t ws_bytes, float *scales, void *stream);

/* gs_loss's value from gs_render_fwd_l1's per-tile sums: loss[3] =
 * (lambda_color Lc + lambda_depth Ld, Lc, Ld), Lc = sum / (3HW), Ld = sum / |V|
 * (0 if |V| = 0), fp64, fixed-order (bit-deterministic; equal to gs_loss's up
 * to the fp64 summation order).  loss_part (device) [T][2]; scales (device)
 * [4] from gs_loss_scales; loss (device) [3]. */
int gs_loss_from_tiles(gs_camera cam, const double *loss_part, const float *scales, float lambda_color,
                       float lambda_depth, float *loss, void *stream);

/* NEXT(1) — masked tracking loss (Eq. 15; S:286-294, S:425-438;
 * DESIGN.md R29-R31).  Tracking only: gradients flow to the rendered colour
 * and depth, the masks are constants (the 3-D Gaussians are frozen).
 *
 *   e_c = (|C^_r - C_r| + |C^_g - C_g| + |C^_b - C_b|) / 3,  e_d = |D^ - D*|
 *         (fp32, each operation rounded to nearest, in this order)
 *   valid pixels: D* > 0;  med_c, med_d = LOWER medians (rank floor((n-1)/2))
 *   of e_c, e_d over the n valid pixels (exact order statistics);
 *   M_inlier = valid & e_d <= fp32(mult med_d) & e_c <= fp32(mult med_c);
 *   M_alpha = alpha^3 (fp32, from the rendered alpha map);
 *   L = sum_px M_inlier M_alpha (lambda_c e_c + (1 - lambda_c) e_d)   (fp64 sum);
 *   dL_dcolor = M_inlier M_alpha (lambda_c / 3) sign(C^ - C*);
 *   dL_ddepth = M_inlier M_alpha (1 - lambda_c) sign(D^ - D*);  sign(0) = 0.
 *   color, depth, alpha (device) rendered maps [3][H][W], [H][W], [H][W]
 *   tgt_color, tgt_depth (device) RGB-D input frame, same layouts
 *   lambda_c in [0, 1]; inlier_mult > 0 (50 in the paper's supplement)
 *   ws     (device) >= gs_tracking_loss_workspace_bytes(cam)
 *   loss   (device) [4] = (L, med_c, med_d, number of inlier pixels); with no
 *          valid pixel every mask is empty and loss = (0, 0, 0, 0)
 * The masks and medians are bit-deterministic; L is a fixed-order reduction.
 * Errors: GS_ERR_INVALID_ARG (null, lambda_c outside [0,1], mult <= 0),
 * GS_ERR_WORKSPACE. */
size_t gs_tracking_loss_workspace_bytes(gs_camera cam);
int gs_tracking_loss(gs_camera cam, const float *color, const float *depth, const float *alpha,
                     const float *tgt_color, const float *tgt_depth, float lambda_c,
                     float inlier_mult, void *ws, size_t ws_bytes, float *loss,
                     float *dL_dcolor, float *dL_ddepth, void *stream);

/* NEXT(2) — SSIM term of the colour loss (Eq. 10: L_color =
 * (1 - lambda) |C^ - C*|_1 + lambda (1 - SSIM(C^, C*)), lambda = 0.2;
 * S:266-274; R32-R33).
 *
 * SSIM per Wang et al. 2004 (the paper's [wang2004image]): per channel and
 * pixel, local means / variances / covariance under an 11x11 Gaussian window
 * (sigma 1.5, normalised) applied as a zero-padded "same" correlation,
 * C1 = 0.01^2, C2 = 0.03^2; SSIM = the mean of the SSIM map over 3HW.
 *   color, tgt_color (device) [3][H][W]
 *   weight   the loss weight w of the SSIM term (lambda_color * lambda)
 *   ws       (device) >= gs_ssim_workspace_bytes(cam)
 *   loss     (device) [4]: loss[0] += w (1 - SSIM), loss[3] = SSIM
 *   dL_dcolor (device) [3][H][W]: += -w dSSIM/dC^ (analytic, through the
 *            local statistics)
 * Call it after gs_loss with lambda_color * (1 - lambda) as gs_loss's colour
 * weight to get Eq. 10 + Eq. 12 (R33).  The SSIM value is a fixed-order
 * reduction (deterministic); the gradient is per-pixel (no atomics).
 * Errors: GS_ERR_INVALID_ARG (null, weight < 0), GS_ERR_WORKSPACE. */
size_t gs_ssim_workspace_bytes(gs_camera cam);
int gs_ssim(gs_camera cam, const float *color, const float *tgt_color, float weight, void *ws,
            size_t ws_bytes, float *loss, float *dL_dcolor, void *stream);

/* NEXT(3) — device epilogue of a mapping iteration ("jointly
 * optimized ... minimizing the loss (12)"; Eq. 11; P:624 pruning;
 * S:205-241; R34-R36).  All calls are asynchronous. */

/* Adam hyper-parameters (host, by pointer).  Learning rates per parameter
 * group (S:231 defaults: mean 1e-4, quaternion 1e-3, log-scale 1e-3, opacity
 * logit 5e-2, colour 2.5e-3; beta 0.9 / 0.999, eps 1e-8); step = t >= 1 (bias
 * correction 1 - beta^t). */
typedef struct {
  float lr_mean, lr_quat, lr_logscale, lr_opacity, lr_rgb;
  double beta1, beta2, eps; /* fp64: 1 - beta is formed without fp32 cancellation */
  int32_t step;
} gs_adam_cfg;

/* Workspace bytes gs_iso_reg / gs_prune need for n Gaussians. */
size_t gs_opt_workspace_bytes(int32_t n);

/* Eq. 11: L_reg = sum_k |s_k - s^bar_k|_1 / |K|, s_k = exp(logscale_k)
 * (3 components), s^bar_k = the mean of s_k's components (R34).
 *   g_logscale (device) [n][4]: += lambda_reg dL_reg/dlogscale (w unused)
 *   loss       (device) [2]: loss[0] += lambda_reg L_reg, loss[1] = L_reg
 * Fixed-order reduction (deterministic). */
int gs_iso_reg(gs_params p, float lambda_reg, float *g_logscale, void *ws, size_t ws_bytes,
               float *loss, void *stream);

/* One Adam step over the four parameter arrays of p, IN PLACE (the arrays of
 * p are written although gs_params declares them const): per component
 * m = b1 m + (1 - b1) g, v = b2 v + (1 - b2) g^2, p -= lr (m / (1 - b1^t)) /
 * (sqrt(v / (1 - b2^t)) + eps); quaternions renormalised after the step
 * (S:220); a Gaussian with any non-finite gradient is left untouched and
 * counted in cnt->n_nonfinite.
 *   g_*      (device) [n][4] gradients (gs_render_bwd's layout)
 *   moments  (device) [n][8][4]: m of (mean_opa, quat, logscale, rgb), then
 *            v; zero-initialise (new Gaussians start from zero)
 *   cnt      (device, nullable) */
int gs_adam_step(gs_params p, const float *g_mean_opa, const float *g_quat,
                 const float *g_logscale, const float *g_rgb, float *moments,
                 const gs_adam_cfg *cfg, gs_counters *cnt, void *stream);

/* Opacity pruning ("prune Gaussians having opacity values lower than a
 * threshold o_thre"): keeps the Gaussians with sigmoid(logit) >= o_thre
 * (decided in fp64, R35), compacted in their original order into `out`
 * (and their moments into moments_out when moments != NULL); *n_out (device)
 * = the kept count.  out / moments_out must not alias the inputs.
 *   ws (device) >= gs_opt_workspace_bytes(p.n) */
int gs_prune(gs_params p, const float *moments, float o_thre, gs_params out,
             float *moments_out, void *ws, size_t ws_bytes, int32_t *n_out, void *stream);

/* NEXT(4) — sub-map seeding from a keyframe ("we sample M_k points
 * uniformly from the regions with the rendered alpha values lower than a
 * threshold alpha_n ... that have no neighbors within a search radius rho
 * ... scales ... based on the nearest neighbor distance"; P:230 alpha_n = 0.6,
 * rho = 0.01 m; P:624 opacity 0.5; R37-R41).
 *
 *   candidates: the first max_new pixels with depth > 0 and alpha < alpha_n in
 *     the order of the seeded bijective permutation of the pixel indices of
 *     R38 (oracle/seed.py writes it out);
 *   points: p_c = ((i - cx) D / fx, (j - cy) D / fy, D), world = R^T (p_c - t)
 *     in fp64, rounded to fp32;
 *   a candidate is rejected if an existing mean or an earlier candidate lies
 *     within rho (squared fp64 distance < rho^2);
 *   accepted points are appended at p.mean_opa / quat / logscale / rgb
 *     [n, n + n_new) in sample order: mean, opacity logit 0 (o = 0.5),
 *     rotation (1, 0, 0, 0), log-scales ln(clamp(nearest-neighbour distance
 *     among existing + accepted points, rho / 2, 0.1 m)), colour of the pixel.
 *   view_host (host) T_wc of the keyframe
 *   color, depth, alpha (device) the keyframe RGB-D and the rendered alpha
 *   capacity  length of the parameter arrays (appends beyond it are dropped;
 *             *n_new still counts them)
 *   n_new     (device) [1] accepted count
 *   ws        (device) >= gs_seed_workspace_bytes(cam, p.n, max_new)
 * Deterministic for a given seed.  Errors: GS_ERR_INVALID_ARG (null, rho
 * not in (0, 0.1], capacity < n), GS_ERR_WORKSPACE. */
size_t gs_seed_workspace_bytes(gs_camera cam, int32_t n, int32_t max_new);
int gs_seed(gs_camera cam, const gs_view *view_host, const float *color, const float *depth,
            const float *alpha, float alpha_n, float rho, int32_t max_new, uint32_t seed,
            gs_params p, int32_t capacity, void *ws, size_t ws_bytes, int32_t *n_new, void *stream);

/* First keyframe of a sub-map, M_c batch ("M_c points from the
 * keyframe point cloud in high color gradient regions"; R43): the
 * high-colour-gradient candidate set as a pseudo-alpha map for gs_seed
 * (alpha_n = 0.5 then samples exactly that set):
 *   grey = (0.299 r + 0.587 g) + 0.114 b, 3x3 Sobel gx, gy on interior
 *   pixels (0 on the border), m2 = gx^2 + gy^2, all IEEE fp64 in this order;
 *   t = the nearest-rank q-percentile of m2 over all pixels (the
 *   ceil(q HW)-th smallest, exact); pseudo_alpha = 0 where m2 > t and
 *   depth > 0, else 1.
 *   color [3][H][W], depth [H][W] (device) the keyframe
 *   q             in (0, 1] (0.95)
 *   pseudo_alpha  (device) [H][W] written
 *   threshold_m2  (device, nullable) [1] fp64: t
 *   ws (device, 8-byte aligned) >= gs_gradient_mask_workspace_bytes(cam)
 * The M_u batch is gs_seed with the empty sub-map's alpha (all 0); the M_c
 * batch then runs against the sub-map holding the M_u Gaussians. */
size_t gs_gradient_mask_workspace_bytes(gs_camera cam);
int gs_gradient_mask(gs_camera cam, const float *color, const float *depth, double q,
                     float *pseudo_alpha, double *threshold_m2, void *ws, size_t ws_bytes,
                     void *stream);

/* Input frames ("the RGBD frame", "the input color and depth map
 * at frame i", "an RGBD sensor"): unpacks a frame in the sensors' and
 * datasets' format, 8-bit RGB and 16-bit depth, into the fp32 planar targets
 * of gs_loss / gs_tracking_loss / gs_seed:
 *   tgt_color[c][q] = rgb[q][c] / 255   (IEEE fp32 division)
 *   tgt_depth[q]    = depth16[q] * depth_scale   (fp32; 0 stays 0 = invalid)
 *   rgb        (device) [H][W][3] uint8, interleaved
 *   depth16    (device) [H][W] uint16, in units of depth_scale metres
 *              (e.g. 1/5000 for TUM-RGBD, 1/6553.5 for Replica)
 *   tgt_color  (device) [3][H][W] fp32;  tgt_depth (device) [H][W] fp32
 *   scales     (device, nullable) [4]: also written as gs_loss_scales(cam,
 *              tgt_depth, lambda_color, lambda_depth) would (the valid-depth
 *              count taken during the unpacking, no second pass)
 * Errors: GS_ERR_INVALID_ARG (null, bad camera, depth_scale <= 0, negative
 * lambdas with scales). */
int gs_unpack_rgbd(gs_camera cam, const uint8_t *rgb, const uint16_t *depth16, float depth_scale,
                   float *tgt_color, float *tgt_depth, float *scales, float lambda_color,
                   float lambda_depth, void *stream);

/* S5+S6 — backward (Eqs. 7-8; R16, R17).
 *
 * Per pixel, replays the composited entries back to front (same alpha
 * decisions as gs_render_fwd, bit for bit) with suffix accumulators
 * (Eq. 8 form), reduces per-Gaussian 2-D gradients (u, v, A, B, C, logit,
 * r, g, b, p_z) with warp shuffles before global atomics, then chains them
 * to the 3-D parameters.
 *   tile_order (device, nullable) from gs_bin_sort: launch order of the tiles
 *   dL_dcolor [3][H][W], dL_ddepth [H][W] (device); dL_dalpha [H][W]
 *             (device, nullable = 0)
 *   flags     GS_GRAD_PARAMS and/or GS_GRAD_POSE, optionally one of
 *             GS_BWD_PIXELS_ONLY (accumulate grad2d only; it then holds the
 *             2-D gradients) / GS_BWD_GAUSS_ONLY (chain an accumulated grad2d
 *             and re-zero it); the two split calls equal one full call;
 *             GS_BWD_ATOMIC_ACC: the += into g_* below is an atomic add, so
 *             per-view calls on different streams need no ordering
 *   ws        (device) >= gs_bwd_workspace_bytes(n), zero on entry
 *   g_mean_opa, g_quat, g_logscale, g_rgb (device) [n][4], ACCUMULATED (+=)
 *             in the layout of gs_params; required iff GS_GRAD_PARAMS
 *   pose_partials (device) [gs_pose_partials_count(n)][12] =
 *             (dL/dR row-major 9, dL/dt 3) per block; required iff
 *             GS_GRAD_POSE, overwritten.
 *   tile_done (device, nullable) the [T + 1] flags given to the immediately
 *             preceding gs_render_fwd_l1 on this stream: the per-pixel phase
 *             is launched as a programmatic dependent of that forward (PDL)
 *             and each tile waits for its forward tile's flag, then re-arms
 *             it.  The wait is capped (~0.4 s): a wait that times out is
 *             counted in tile_done[T] and its flag is NOT re-armed, so a
 *             broken ordering is never silent (the results of that call are
 *             invalid; TrackingLoop.flag_timeouts() reads the count).  NULL:
 *             ordinary stream order. */
int gs_render_bwd(gs_params p, const gs_view *view, gs_camera cam, gs_proj pr,
                  const int32_t *sorted_idx, const int32_t *tile_range,
                  const int32_t *tile_order, const float *T_final, const int32_t *n_contrib,
                  const float *dL_dcolor, const float *dL_ddepth,
                  const float *dL_dalpha, uint32_t flags, void *ws, size_t ws_bytes,
                  float *g_mean_opa, float *g_quat, float *g_logscale, float *g_rgb,
                  float *pose_partials, uint32_t *tile_done, void *stream);

/* S7 — camera-pose gradient (Eq. 14; R22).
 *
 * Reduces the pose partials in a fixed order to dL/dR, dL/dt and converts
 * them to the left-perturbation twist xi = (v, w) (T <- exp(xi^) T) and to
 * the (q, t) parameterisation of T_wc (q = (w, x, y, z)).
 *   view          (device) T_wc; updated in place iff step != NULL:
 *                 Adam on the twist, T <- exp(-step^) T, R re-orthonormalised
 *   pose_partials (device) [n_partials][12]
 *   step          (host, nullable) Adam hyper-parameters
 *   adam_state    (device) [13] fp64 = m[6], v[6], t; required iff step !=
 *                 NULL; zero it before the first iteration (the moments are
 *                 kept in fp64, so the step equals the fp64 definition up to
 *                 the fp32 rounding of the stored view)
 *   dL_dview      (device, nullable) [12] = dL/dR (9), dL/dt (3)
 *   dL_dtwist     (device, nullable) [6]  = dL/dv (3), dL/dw (3)
 *   dL_dqt        (device, nullable) [7]  = dL/dq (4), dL/dt (3) */
int gs_pose_grad(gs_view *view, const float *pose_partials, int32_t n_partials,
                 const gs_pose_step *step, double *adam_state, float *dL_dview,
                 float *dL_dtwist, float *dL_dqt, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* GS_H */
