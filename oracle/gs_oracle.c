/*
 * gs_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the
 * differentiable Gaussian-splatting rasterizer of Gaussian-SLAM
 * (arXiv 2312.10070, "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
 * readings R1..R26 = DESIGN.md §3 / SURVEY §8(c)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header,
 * constant or helper with the CUDA path (paper_2312_10070_b200/csrc), and the
 * CUDA path never loads it.
 *
 * fp32 inputs are promoted exactly to fp64; every computation below is fp64.
 * Build: gcc -O2 -fopenmp -ffp-contract=off (no FMA contraction, so the
 * decision path (R1) has one documented rounding order).
 *
 * Parity status: every function is pinned by tests in
 * tests/test_oracle_*.py (closed forms, invariants, library routines, brute
 * force, central finite differences).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Rasterizer constants, as the fp32 values the method uses (R11, R7). */
#define OR_TILE 16
static const double OR_DILATION = (double)0.3f;
static const double OR_ALPHA_MAX = (double)0.999f;
static const double OR_ALPHA_MIN = (double)(1.0f / 255.0f);
static const double OR_T_EPS = (double)1e-4f;

/* Camera as double[8] = (W, H, fx, fy, cx, cy, z_near, z_far). */
typedef struct {
  int W, H, TX, TY;
  double fx, fy, cx, cy, znear, zfar;
} ocam;

static ocam mkcam(const double *c) {
  ocam k;
  k.W = (int)c[0];
  k.H = (int)c[1];
  k.fx = c[2];
  k.fy = c[3];
  k.cx = c[4];
  k.cy = c[5];
  k.znear = c[6];
  k.zfar = c[7];
  k.TX = (k.W + OR_TILE - 1) / OR_TILE;
  k.TY = (k.H + OR_TILE - 1) / OR_TILE;
  return k;
}

int or_num_tiles(const double *cam) {
  ocam k = mkcam(cam);
  return k.TX * k.TY;
}

/* ------------------------------------------------------------------ */
/* Geometry ("Covariance is decomposed as Sigma = R S S^T R^T"; */
/* S:47-64).                                                            */

/* Rotation matrix of a unit quaternion (w, x, y, z). */
void or_quat_to_rot(const double *q, double *Rq) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  Rq[0] = 1.0 - 2.0 * (y * y + z * z);
  Rq[1] = 2.0 * (x * y - w * z);
  Rq[2] = 2.0 * (x * z + w * y);
  Rq[3] = 2.0 * (x * y + w * z);
  Rq[4] = 1.0 - 2.0 * (x * x + z * z);
  Rq[5] = 2.0 * (y * z - w * x);
  Rq[6] = 2.0 * (x * z - w * y);
  Rq[7] = 2.0 * (y * z + w * x);
  Rq[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* Sigma = (R_q S)(R_q S)^T with S = diag(exp(logscale)). */
void or_covariance(const double *q_in, const double *logscale, double *Sigma) {
  double qn = sqrt(((q_in[0] * q_in[0] + q_in[1] * q_in[1]) + q_in[2] * q_in[2]) +
                   q_in[3] * q_in[3]);
  double q[4] = {q_in[0] / qn, q_in[1] / qn, q_in[2] / qn, q_in[3] / qn};
  double Rq[9], M[9];
  or_quat_to_rot(q, Rq);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) M[3 * i + k] = Rq[3 * i + k] * exp(logscale[k]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      Sigma[3 * i + j] = (M[3 * i + 0] * M[3 * j + 0] + M[3 * i + 1] * M[3 * j + 1]) +
                         M[3 * i + 2] * M[3 * j + 2];
}

/* ------------------------------------------------------------------ */
/* S1 projection (Eqs. 1-2).                      */

/* Per-Gaussian intermediate quantities, recomputed by the backward. */
typedef struct {
  int culled; /* 0 visible; 1 near/far; 2 non-finite/singular; 3 off-screen */
  double q[4];   /* normalised quaternion */
  double qn;     /* |q| */
  double Rq[9];  /* R(q^) */
  double s[3];   /* exp(logscale) */
  double M[9];   /* R_q S */
  double Sig[9]; /* Sigma (world) */
  double p[3];   /* camera-frame mean */
  double J[6];   /* 2x3 perspective Jacobian */
  double Sc[9];  /* R Sigma R^T */
  double a, b, c; /* Sigma^I + 0.3 I = [[a, b], [b, c]] */
  double det, A, B, C; /* conic = inverse */
  double u, v;
  double hx, hy; /* half-widths of the alpha >= 1/255 box (R8') */
  int rect[4];
  double o;
} ogauss;

static void project_one(const double *mu, const double *qin, const double *ls, double logit,
                        const double *R, const double *t, const ocam *k, ogauss *g) {
  memset(g, 0, sizeof(*g));
  g->rect[2] = -1;
  g->rect[3] = -1;
  /* q^ = q/|q| (R18) */
  g->qn = sqrt(((qin[0] * qin[0] + qin[1] * qin[1]) + qin[2] * qin[2]) + qin[3] * qin[3]);
  for (int i = 0; i < 4; ++i) g->q[i] = qin[i] / g->qn;
  or_quat_to_rot(g->q, g->Rq);
  for (int i = 0; i < 3; ++i) g->s[i] = exp(ls[i]);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) g->M[3 * i + j] = g->Rq[3 * i + j] * g->s[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      g->Sig[3 * i + j] = (g->M[3 * i + 0] * g->M[3 * j + 0] + g->M[3 * i + 1] * g->M[3 * j + 1]) +
                          g->M[3 * i + 2] * g->M[3 * j + 2];
  /* p = R mu + t: the world-to-camera transform T_wc of Eq. 1 */
  for (int i = 0; i < 3; ++i)
    g->p[i] = ((R[3 * i + 0] * mu[0] + R[3 * i + 1] * mu[1]) + R[3 * i + 2] * mu[2]) + t[i];
  g->o = 1.0 / (1.0 + exp(-logit)); /* opacity = sigmoid(logit) (R18) */
  double x = g->p[0], y = g->p[1], z = g->p[2];
  if (!isfinite(x) || !isfinite(y) || !isfinite(z) || !isfinite(g->qn) || !(g->qn > 0.0)) {
    g->culled = 2;
    return;
  }
  if (!(z >= k->znear && z <= k->zfar)) { /* near/far cull (R5) */
    g->culled = 1;
    return;
  }
  /* pinhole pi (R4): u = fx x/z + cx */
  g->u = (k->fx * x) / z + k->cx;
  g->v = (k->fy * y) / z + k->cy;
  /* EWA Jacobian, unclamped (Eq. 2 "affine transformation from [zwicker]", R6) */
  double z2 = z * z;
  g->J[0] = k->fx / z;
  g->J[1] = 0.0;
  g->J[2] = -(k->fx * x) / z2;
  g->J[3] = 0.0;
  g->J[4] = k->fy / z;
  g->J[5] = -(k->fy * y) / z2;
  /* Sigma_c = R Sigma R^T (Eq. 2: R_wc Sigma R_wc^T) */
  double W[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      W[3 * i + j] = (R[3 * i + 0] * g->Sig[0 + j] + R[3 * i + 1] * g->Sig[3 + j]) +
                     R[3 * i + 2] * g->Sig[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      g->Sc[3 * i + j] = (W[3 * i + 0] * R[3 * j + 0] + W[3 * i + 1] * R[3 * j + 1]) +
                         W[3 * i + 2] * R[3 * j + 2];
  /* Sigma^I = J Sigma_c J^T (Eq. 2), with J01 = J10 = 0 */
  double T0[3], T1[3];
  for (int j = 0; j < 3; ++j) {
    T0[j] = g->J[0] * g->Sc[0 + j] + g->J[2] * g->Sc[6 + j];
    T1[j] = g->J[4] * g->Sc[3 + j] + g->J[5] * g->Sc[6 + j];
  }
  double s00 = T0[0] * g->J[0] + T0[2] * g->J[2];
  double s01 = T0[1] * g->J[4] + T0[2] * g->J[5];
  double s11 = T1[1] * g->J[4] + T1[2] * g->J[5];
  /* low-pass dilation +0.3 px^2 (R7) */
  g->a = s00 + OR_DILATION;
  g->b = s01;
  g->c = s11 + OR_DILATION;
  g->det = g->a * g->c - g->b * g->b;
  if (!(g->det > 0.0) || !isfinite(g->det) || !isfinite(g->u) || !isfinite(g->v)) {
    g->culled = 2; /* singular Sigma^I */
    return;
  }
  g->A = g->c / g->det;
  g->B = -g->b / g->det;
  g->C = g->a / g->det;
  /* tile membership (R8'): the tiles meeting the axis-aligned box of the region
   * where alpha~ = o exp(-sigma) >= 1/255, i.e. sigma <= tau = ln(o / alpha_min):
   * the ellipse Delta^T (Sigma^I)^-1 Delta <= 2 tau, whose half-widths are
   * sqrt(2 tau a) and sqrt(2 tau c).  A Gaussian whose alpha~ never reaches
   * 1/255 (tau <= 0) touches no tile. */
  double tau = log(g->o / OR_ALPHA_MIN);
  if (!(tau > 0.0)) {
    g->culled = 3;
    return;
  }
  g->hx = sqrt((2.0 * tau) * g->a);
  g->hy = sqrt((2.0 * tau) * g->c);
  int x0 = (int)floor((g->u - g->hx) / OR_TILE), x1 = (int)floor((g->u + g->hx) / OR_TILE);
  int y0 = (int)floor((g->v - g->hy) / OR_TILE), y1 = (int)floor((g->v + g->hy) / OR_TILE);
  if (x0 < 0) x0 = 0;
  if (y0 < 0) y0 = 0;
  if (x1 > k->TX - 1) x1 = k->TX - 1;
  if (y1 > k->TY - 1) y1 = k->TY - 1;
  if (x0 > x1 || y0 > y1) {
    g->culled = 3;
    return;
  }
  g->rect[0] = x0;
  g->rect[1] = y0;
  g->rect[2] = x1;
  g->rect[3] = y1;
}

/* Public projection.  Arrays: mean[n][3], quat[n][4], logscale[n][3],
 * logit[n], R[9], t[3], cam[8].  Outputs (nullable each): uv[n][2],
 * conic[n][3] (A, B, C), opac[n], pz[n], depth_key[n] (fp32 RN(p_z), +inf if
 * culled), hxy[n][2] (half-widths of the alpha >= 1/255 box), rect[n][4],
 * culled[n], cov2d[n][3] (a, b, c). */
void or_project(int n, const double *mean, const double *quat, const double *logscale,
                const double *logit, const double *R, const double *t, const double *cam,
                double *uv, double *conic, double *opac, double *pz, float *depth_key,
                double *hxy, int *rect, int *culled, double *cov2d) {
  ocam k = mkcam(cam);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    ogauss g;
    project_one(mean + 3 * i, quat + 4 * i, logscale + 3 * i, logit[i], R, t, &k, &g);
    if (uv) { uv[2 * i] = g.u; uv[2 * i + 1] = g.v; }
    if (conic) { conic[3 * i] = g.A; conic[3 * i + 1] = g.B; conic[3 * i + 2] = g.C; }
    if (opac) opac[i] = g.o;
    if (pz) pz[i] = g.p[2];
    if (depth_key) depth_key[i] = g.culled ? INFINITY : (float)g.p[2];
    if (hxy) { hxy[2 * i] = g.culled ? 0.0 : g.hx; hxy[2 * i + 1] = g.culled ? 0.0 : g.hy; }
    if (rect) for (int j = 0; j < 4; ++j) rect[4 * i + j] = g.rect[j];
    if (culled) culled[i] = g.culled;
    if (cov2d) { cov2d[3 * i] = g.a; cov2d[3 * i + 1] = g.b; cov2d[3 * i + 2] = g.c; }
  }
}

/* ------------------------------------------------------------------ */
/* S2 binning ("m ordered Gaussians"; R10).          */

typedef struct {
  float key;
  int idx;
} okey;

static int cmp_key(const void *pa, const void *pb) {
  const okey *a = (const okey *)pa, *b = (const okey *)pb;
  if (a->key < b->key) return -1;
  if (a->key > b->key) return 1;
  return (a->idx > b->idx) - (a->idx < b->idx);
}

/* Count pairs: sum over visible Gaussians of their rect area. */
int64_t or_count_pairs(int n, const int *rect, const int *culled) {
  int64_t P = 0;
  for (int i = 0; i < n; ++i)
    if (!culled[i]) P += (int64_t)(rect[4 * i + 2] - rect[4 * i + 0] + 1) * (rect[4 * i + 3] - rect[4 * i + 1] + 1);
  return P;
}

/* For each tile, the visible Gaussians whose rect contains it, ordered by
 * (fp32 depth key asc, index asc); tiles concatenated in tile-id order.
 * sorted_idx[P] (P from or_count_pairs), tile_range[T][2]. */
void or_bin(int n, const double *cam, const int *rect, const int *culled,
            const float *depth_key, int *sorted_idx, int *tile_range) {
  ocam k = mkcam(cam);
  int T = k.TX * k.TY;
  int64_t *cnt = (int64_t *)calloc((size_t)T + 1, sizeof(int64_t));
  for (int i = 0; i < n; ++i) {
    if (culled[i]) continue;
    for (int ty = rect[4 * i + 1]; ty <= rect[4 * i + 3]; ++ty)
      for (int tx = rect[4 * i + 0]; tx <= rect[4 * i + 2]; ++tx) cnt[ty * k.TX + tx + 1]++;
  }
  for (int t = 0; t < T; ++t) cnt[t + 1] += cnt[t];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
  for (int t = 0; t < T; ++t) fill[t] = cnt[t];
  okey *keys = (okey *)malloc(sizeof(okey) * (size_t)(cnt[T] > 0 ? cnt[T] : 1));
  for (int i = 0; i < n; ++i) {
    if (culled[i]) continue;
    for (int ty = rect[4 * i + 1]; ty <= rect[4 * i + 3]; ++ty)
      for (int tx = rect[4 * i + 0]; tx <= rect[4 * i + 2]; ++tx) {
        int64_t p = fill[ty * k.TX + tx]++;
        keys[p].key = depth_key[i];
        keys[p].idx = i;
      }
  }
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = 0; t < T; ++t) qsort(keys + cnt[t], (size_t)(cnt[t + 1] - cnt[t]), sizeof(okey), cmp_key);
  for (int64_t p = 0; p < cnt[T]; ++p) sorted_idx[p] = keys[p].idx;
  for (int t = 0; t < T; ++t) {
    tile_range[2 * t] = (int)cnt[t];
    tile_range[2 * t + 1] = (int)cnt[t + 1];
  }
  free(keys);
  free(fill);
  free(cnt);
}

/* ------------------------------------------------------------------ */
/* S3 forward compositing (Eqs. 3, 4, 6). */

/* alpha of Gaussian g at pixel (px, py): Eq. 4, alpha = o exp(-sigma),
 * sigma = 1/2 Delta^T (Sigma^I)^-1 Delta, Delta = mu^I - pixel (R3). */
static double alpha_tilde(const double *uv, const double *conic, double o, double px, double py,
                          double *dx_out, double *dy_out) {
  double dx = uv[0] - px, dy = uv[1] - py;
  double sigma = 0.5 * (conic[0] * dx * dx + 2.0 * conic[1] * dx * dy + conic[2] * dy * dy);
  if (dx_out) { *dx_out = dx; *dy_out = dy; }
  return o * exp(-sigma);
}

static double rel_margin(double x, double thr) { return fabs(x - thr) / thr; }

/* Per-pixel forward. Outputs (planar): color[3][H][W], depth, alpha, Tfinal,
 * n_contrib (tile-list position of the last composited entry + 1), scanned,
 * contrib (counts), margin (min relative decision margin, R2), sig (64-bit
 * hash of the composited (position, clamp) sequence; H8 decision signature).
 * tile_mask[T] (nullable): render only tiles with tile_mask != 0. */
void or_render(int n, const double *cam, const double *uv, const double *conic,
               const double *opac, const double *pz, const double *rgb,
               const int *sorted_idx, const int *tile_range, const unsigned char *tile_mask,
               double *color, double *depth, double *alpha, double *Tfinal, int *n_contrib,
               int *scanned, int *contrib, double *margin, uint64_t *sig) {
  ocam k = mkcam(cam);
  int T = k.TX * k.TY;
  size_t HW = (size_t)k.W * k.H;
  (void)n;
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < T; ++t) {
    if (tile_mask && !tile_mask[t]) continue;
    int tx = t % k.TX, ty = t / k.TX;
    int s0 = tile_range[2 * t], s1 = tile_range[2 * t + 1];
    for (int py = ty * OR_TILE; py < (ty + 1) * OR_TILE && py < k.H; ++py)
      for (int px = tx * OR_TILE; px < (tx + 1) * OR_TILE && px < k.W; ++px) {
        double Tr = 1.0, C[3] = {0, 0, 0}, D = 0.0, Aacc = 0.0, mg = INFINITY;
        int last = 0, nscan = 0, ncon = 0;
        uint64_t h = 1469598103934665603ull;
        for (int p = s0; p < s1; ++p) {
          int g = sorted_idx[p];
          double at = alpha_tilde(uv + 2 * g, conic + 3 * g, opac[g], px, py, NULL, NULL);
          nscan++;
          double m1 = rel_margin(at, OR_ALPHA_MIN);
          double m2 = rel_margin(at, OR_ALPHA_MAX);
          if (m1 < mg) mg = m1;
          if (m2 < mg) mg = m2;
          double a = at < OR_ALPHA_MAX ? at : OR_ALPHA_MAX; /* clamp (R11) */
          if (a < OR_ALPHA_MIN) continue;                   /* skip (R11) */
          double w = a * Tr;                                /* alpha_j T_j */
          for (int ch = 0; ch < 3; ++ch) C[ch] += rgb[3 * g + ch] * w; /* Eq. 3 */
          D += pz[g] * w;                                             /* Eq. 6 */
          Aacc += w;                                                  /* R14 */
          Tr = Tr * (1.0 - a);
          ncon++;
          last = p - s0 + 1;
          h = (h ^ (uint64_t)(p - s0 + 1)) * 1099511628211ull;
          h = (h ^ (uint64_t)(at >= OR_ALPHA_MAX)) * 1099511628211ull;
          double m3 = rel_margin(Tr, OR_T_EPS);
          if (m3 < mg) mg = m3;
          if (Tr < OR_T_EPS) break; /* include, then stop (R11) */
        }
        size_t q = (size_t)py * k.W + px;
        for (int ch = 0; ch < 3; ++ch) color[ch * HW + q] = C[ch];
        depth[q] = D;
        alpha[q] = Aacc;
        Tfinal[q] = Tr;
        n_contrib[q] = last;
        if (scanned) scanned[q] = nscan;
        if (contrib) contrib[q] = ncon;
        if (margin) margin[q] = mg;
        if (sig) sig[q] = h;
      }
  }
}

/* ------------------------------------------------------------------ */
/* S4 loss (Eqs. 9, 10 (L1 part), 12; R20, R21).     */

static double sgn(double x) { return (x > 0.0) - (x < 0.0); }

/* out_loss[3] = (lc*Lc + ld*Ld, Lc, Ld); gradient maps.  weight nullable. */
void or_loss(const double *cam, const double *color, const double *depth, const double *tc,
             const double *td, const double *weight, double lc, double ld, double *out_loss,
             double *g_color, double *g_depth) {
  ocam k = mkcam(cam);
  size_t HW = (size_t)k.W * k.H;
  double sc = 0.0, sd = 0.0;
  int64_t nv = 0;
  for (size_t q = 0; q < HW; ++q)
    if (td[q] > 0.0) nv++;
  for (size_t q = 0; q < HW; ++q) {
    double w = weight ? weight[q] : 1.0;
    for (int ch = 0; ch < 3; ++ch) {
      double r = color[ch * HW + q] - tc[ch * HW + q];
      sc += w * fabs(r);
      g_color[ch * HW + q] = lc * w * sgn(r) / (3.0 * (double)HW);
    }
    if (td[q] > 0.0) {
      double r = depth[q] - td[q];
      sd += w * fabs(r);
      g_depth[q] = ld * w * sgn(r) / (double)nv;
    } else {
      g_depth[q] = 0.0;
    }
  }
  double Lc = sc / (3.0 * (double)HW);
  double Ld = nv > 0 ? sd / (double)nv : 0.0;
  out_loss[0] = lc * Lc + ld * Ld;
  out_loss[1] = Lc;
  out_loss[2] = Ld;
}

/* ------------------------------------------------------------------ */
/* S5 backward, per pixel (Eqs. 7-8).              */
/* 2-D quantities per Gaussian, in this order:                           */
/*   0 u, 1 v, 2 A, 3 B, 4 C, 5 opacity logit, 6 r, 7 g, 8 b, 9 p_z        */
#define NG2 10

/* Per-pair accumulators are summed per tile by one thread, then reduced per
 * Gaussian in pair order: deterministic.  m2 = sum of |contribution| with
 * every inner sum expanded in absolute value (the magnitude scale of R23). */
static void bwd_pixels(const ocam *k, const double *uv, const double *conic, const double *opac,
                       const double *pz, const double *rgb, const int *sorted_idx,
                       const int *tile_range, const unsigned char *tile_mask, const double *gC,
                       const double *gD, const double *gA, double *pair_g, double *pair_m) {
  int T = k->TX * k->TY;
  size_t HW = (size_t)k->W * k->H;
#pragma omp parallel
  {
    int cap = 0;
    double *al = NULL, *at_ = NULL, *Tj = NULL;
    int *pos = NULL;
#pragma omp for schedule(dynamic, 1)
    for (int t = 0; t < T; ++t) {
      if (tile_mask && !tile_mask[t]) continue;
      int tx = t % k->TX, ty = t / k->TX;
      int s0 = tile_range[2 * t], s1 = tile_range[2 * t + 1];
      int len = s1 - s0;
      if (len > cap) {
        cap = len;
        al = (double *)realloc(al, sizeof(double) * cap);
        at_ = (double *)realloc(at_, sizeof(double) * cap);
        Tj = (double *)realloc(Tj, sizeof(double) * cap);
        pos = (int *)realloc(pos, sizeof(int) * cap);
      }
      for (int py = ty * OR_TILE; py < (ty + 1) * OR_TILE && py < k->H; ++py)
        for (int px = tx * OR_TILE; px < (tx + 1) * OR_TILE && px < k->W; ++px) {
          size_t q = (size_t)py * k->W + px;
          /* forward replay: the composited list m (Eq. 3) with alpha_j, T_j */
          int m = 0;
          double Tr = 1.0;
          for (int p = s0; p < s1; ++p) {
            int g = sorted_idx[p];
            double a_t = alpha_tilde(uv + 2 * g, conic + 3 * g, opac[g], px, py, NULL, NULL);
            double a = a_t < OR_ALPHA_MAX ? a_t : OR_ALPHA_MAX;
            if (a < OR_ALPHA_MIN) continue;
            al[m] = a;
            at_[m] = a_t;
            Tj[m] = Tr;
            pos[m] = p;
            m++;
            Tr = Tr * (1.0 - a);
            if (Tr < OR_T_EPS) break;
          }
          double G[3] = {gC[q], gC[HW + q], gC[2 * HW + q]};
          double Gd = gD[q], Ga = gA ? gA[q] : 0.0;
          /* suffix sums sum_{u>j} X_u alpha_u T_u of Eq. 8, X = c (3), z, 1 */
          double sufC[3] = {0, 0, 0}, sufD = 0.0, sufA = 0.0;
          double asufC[3] = {0, 0, 0}, asufD = 0.0, asufA = 0.0; /* |.| versions */
          for (int j = m - 1; j >= 0; --j) {
            int p = pos[j], g = sorted_idx[p];
            double a = al[j], T_ = Tj[j];
            const double *c = rgb + 3 * g;
            double z = pz[g];
            double inv1ma = 1.0 / (1.0 - a);
            /* Eq. 8: dD/dalpha_j = z_j T_j - sum_{u>j} z_u alpha_u T_u / (1 - alpha_j);
             * "the gradients for [colour] ... are computed similarly" */
            double dCda[3], dDda, dAda, adCda[3], adDda, adAda;
            for (int ch = 0; ch < 3; ++ch) {
              dCda[ch] = c[ch] * T_ - sufC[ch] * inv1ma;
              adCda[ch] = fabs(c[ch]) * T_ + fabs(asufC[ch]) * inv1ma;
            }
            dDda = z * T_ - sufD * inv1ma;
            adDda = fabs(z) * T_ + asufD * inv1ma;
            dAda = T_ - sufA * inv1ma;
            adAda = T_ + asufA * inv1ma;
            /* chain rule, Eq. 7: dL/dalpha_j = sum_i dL/dX_i dX_i/dalpha_j */
            double galpha = (G[0] * dCda[0] + G[1] * dCda[1] + G[2] * dCda[2]) + Gd * dDda + Ga * dAda;
            double agalpha = (fabs(G[0]) * adCda[0] + fabs(G[1]) * adCda[1] + fabs(G[2]) * adCda[2]) +
                             fabs(Gd) * adDda + fabs(Ga) * adAda;
            double w = a * T_;
            double *pg = pair_g + (size_t)p * NG2, *pm = pair_m + (size_t)p * NG2;
            for (int ch = 0; ch < 3; ++ch) { /* dC/dc_j = alpha_j T_j */
              pg[6 + ch] += G[ch] * w;
              pm[6 + ch] += fabs(G[ch] * w);
            }
            pg[9] += Gd * w; /* dD/dz_j = alpha_j T_j */
            pm[9] += fabs(Gd * w);
            if (at_[j] < OR_ALPHA_MAX) { /* clamped alpha has no gradient (R17) */
              double dx, dy;
              int gg = g;
              double a_t = alpha_tilde(uv + 2 * gg, conic + 3 * gg, opac[gg], px, py, &dx, &dy);
              (void)a_t;
              double o = opac[g];
              /* alpha = o exp(-sigma): dalpha/dlogit = alpha (1 - o), dalpha/dsigma = -alpha */
              pg[5] += galpha * a * (1.0 - o);
              pm[5] += agalpha * a * (1.0 - o);
              double gsig = -a * galpha, agsig = a * agalpha;
              const double *cn = conic + 3 * g;
              /* sigma = 1/2 (A dx^2 + 2 B dx dy + C dy^2), Delta = mu^I - pixel */
              pg[0] += gsig * (cn[0] * dx + cn[1] * dy);
              pg[1] += gsig * (cn[1] * dx + cn[2] * dy);
              pg[2] += gsig * 0.5 * dx * dx;
              pg[3] += gsig * dx * dy;
              pg[4] += gsig * 0.5 * dy * dy;
              pm[0] += agsig * (fabs(cn[0] * dx) + fabs(cn[1] * dy));
              pm[1] += agsig * (fabs(cn[1] * dx) + fabs(cn[2] * dy));
              pm[2] += agsig * 0.5 * dx * dx;
              pm[3] += agsig * fabs(dx * dy);
              pm[4] += agsig * 0.5 * dy * dy;
            }
            for (int ch = 0; ch < 3; ++ch) {
              sufC[ch] += c[ch] * w;
              asufC[ch] += fabs(c[ch]) * w;
            }
            sufD += z * w;
            asufD += fabs(z) * w;
            sufA += w;
            asufA += w;
          }
        }
    }
    free(al);
    free(at_);
    free(Tj);
    free(pos);
  }
}

/* ------------------------------------------------------------------ */
/* S6 per-Gaussian chain 2-D -> 3-D ("derived as in [kerbl]").      */
/* Linear in g2.  out3[16] in the gs_params layout:                        */
/*   (mu_x, mu_y, mu_z, logit, qw, qx, qy, qz, ls_x, ls_y, ls_z, 0, r, g, b, 0) */
/* pose[12] = (dL/dR row-major 9, dL/dt 3) contribution of this Gaussian.   */
static void chain3d(const ogauss *G, const double *mu, const double *R, const ocam *k,
                    const double *g2, double *out3, double *pose) {
  double x = G->p[0], y = G->p[1], z = G->p[2];
  double gu = g2[0], gv = g2[1], gA = g2[2], gB = g2[3], gC = g2[4];
  /* conic -> Sigma^I: G_Sigma = -Conic G_M Conic, G_M = [[gA, gB/2], [gB/2, gC]] */
  double Cn[4] = {G->A, G->B, G->B, G->C};
  double GM[4] = {gA, 0.5 * gB, 0.5 * gB, gC};
  double t1[4], GS2[4];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) t1[2 * i + j] = Cn[2 * i] * GM[j] + Cn[2 * i + 1] * GM[2 + j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) GS2[2 * i + j] = -(t1[2 * i] * Cn[j] + t1[2 * i + 1] * Cn[2 + j]);
  /* Sigma^I = J Sigma_c J^T (+0.3 I, no gradient): G_Sc = J^T G_S2 J, G_J = 2 G_S2 J Sigma_c */
  const double *J = G->J, *Sc = G->Sc;
  double GSc[9], GJ[6], GJ0[6];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) acc += J[3 * i + a] * GS2[2 * i + j] * J[3 * j + b];
      GSc[3 * a + b] = acc;
    }
  for (int i = 0; i < 2; ++i)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int j = 0; j < 2; ++j) acc += GS2[2 * i + j] * J[3 * j + b];
      GJ0[3 * i + b] = acc;
    }
  for (int i = 0; i < 2; ++i)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += GJ0[3 * i + c] * Sc[3 * c + b];
      GJ[3 * i + b] = 2.0 * acc;
    }
  /* camera-frame mean p: through (u, v) (Eq. 1), J(p) and the depth term (Eq. 6) */
  double fx = k->fx, fy = k->fy, z2 = z * z, z3 = z2 * z;
  double gp[3];
  gp[0] = gu * fx / z + GJ[2] * (-fx / z2);
  gp[1] = gv * fy / z + GJ[5] * (-fy / z2);
  gp[2] = gu * (-fx * x / z2) + gv * (-fy * y / z2) + g2[9] + GJ[0] * (-fx / z2) +
          GJ[2] * (2.0 * fx * x / z3) + GJ[4] * (-fy / z2) + GJ[5] * (2.0 * fy * y / z3);
  /* p = R mu + t  =>  dL/dmu = R^T dL/dp */
  for (int i = 0; i < 3; ++i) out3[i] = R[i] * gp[0] + R[3 + i] * gp[1] + R[6 + i] * gp[2];
  out3[3] = g2[5];
  /* Sigma_c = R Sigma R^T  =>  G_Sigma = R^T G_Sc R */
  double tmp[9], GSig[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += R[3 * c + a] * GSc[3 * c + b];
      tmp[3 * a + b] = acc;
    }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += tmp[3 * a + c] * R[3 * c + b];
      GSig[3 * a + b] = acc;
    }
  /* Sigma = M M^T, M = R_q S  =>  G_M = 2 G_Sigma M (G_Sigma symmetric) */
  double GM3[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += (GSig[3 * a + c] + GSig[3 * c + a]) * G->M[3 * c + b];
      GM3[3 * a + b] = acc;
    }
  /* M_ik = Rq_ik s_k: dL/dlogscale_k = s_k sum_i G_M[i][k] Rq[i][k]; G_Rq = G_M S */
  double GRq[9];
  for (int kk = 0; kk < 3; ++kk) {
    double acc = 0.0;
    for (int i = 0; i < 3; ++i) acc += GM3[3 * i + kk] * G->Rq[3 * i + kk];
    out3[8 + kk] = acc * G->s[kk];
  }
  out3[11] = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int kk = 0; kk < 3; ++kk) GRq[3 * i + kk] = GM3[3 * i + kk] * G->s[kk];
  /* R(q^) derivatives, q^ = (w, x, y, z) */
  double w = G->q[0], qx = G->q[1], qy = G->q[2], qz = G->q[3];
  double dw[9] = {0, -2 * qz, 2 * qy, 2 * qz, 0, -2 * qx, -2 * qy, 2 * qx, 0};
  double dx_[9] = {0, 2 * qy, 2 * qz, 2 * qy, -4 * qx, -2 * w, 2 * qz, 2 * w, -4 * qx};
  double dy_[9] = {-4 * qy, 2 * qx, 2 * w, 2 * qx, 0, 2 * qz, -2 * w, 2 * qz, -4 * qy};
  double dz_[9] = {-4 * qz, -2 * w, 2 * qx, 2 * w, -4 * qz, 2 * qy, 2 * qx, 2 * qy, 0};
  double gqh[4] = {0, 0, 0, 0};
  for (int i = 0; i < 9; ++i) {
    gqh[0] += GRq[i] * dw[i];
    gqh[1] += GRq[i] * dx_[i];
    gqh[2] += GRq[i] * dy_[i];
    gqh[3] += GRq[i] * dz_[i];
  }
  /* q^ = q/|q|: dL/dq = (g - q^ (q^ . g)) / |q| (R18) */
  double dot = gqh[0] * w + gqh[1] * qx + gqh[2] * qy + gqh[3] * qz;
  for (int i = 0; i < 4; ++i) out3[4 + i] = (gqh[i] - G->q[i] * dot) / G->qn;
  for (int ch = 0; ch < 3; ++ch) out3[12 + ch] = g2[6 + ch];
  out3[15] = 0.0;
  if (pose) {
    /* pose: p = R mu + t, Sigma_c = R Sigma R^T
     * dL/dt = dL/dp;  dL/dR = dL/dp mu^T + 2 G_Sc R Sigma */
    double RS[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int c = 0; c < 3; ++c) acc += R[3 * a + c] * G->Sig[3 * c + b];
        RS[3 * a + b] = acc;
      }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int c = 0; c < 3; ++c) acc += (GSc[3 * a + c] + GSc[3 * c + a]) * RS[3 * c + b];
        pose[3 * a + b] = gp[a] * mu[b] + acc;
      }
    for (int i = 0; i < 3; ++i) pose[9 + i] = gp[i];
  }
}

/* Full backward.  gC[3][H][W], gD[H][W], gA[H][W] (nullable) upstream maps.
 * Outputs: g2[n][10], m2[n][10] (2-D grads and magnitudes), g3[n][16],
 * m3[n][16] (3-D grads and magnitudes |d x2D/d theta|^T m2), pose[12],
 * mpose[12] (nullable), all overwritten.  tile_mask nullable. */
void or_backward(int n, const double *mean, const double *quat, const double *logscale,
                 const double *logit, const double *rgb, const double *R, const double *t,
                 const double *cam, const int *sorted_idx, const int *tile_range, int64_t P,
                 const unsigned char *tile_mask, const double *gC, const double *gD,
                 const double *gA, double *g2, double *m2, double *g3, double *m3,
                 double *pose, double *mpose) {
  ocam k = mkcam(cam);
  double *uv = (double *)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
  double *conic = (double *)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  double *opac = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *pz = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  or_project(n, mean, quat, logscale, logit, R, t, cam, uv, conic, opac, pz, NULL, NULL, NULL,
             NULL, NULL);
  double *pair_g = (double *)calloc((size_t)(P > 0 ? P : 1) * NG2, sizeof(double));
  double *pair_m = (double *)calloc((size_t)(P > 0 ? P : 1) * NG2, sizeof(double));
  bwd_pixels(&k, uv, conic, opac, pz, rgb, sorted_idx, tile_range, tile_mask, gC, gD, gA, pair_g,
             pair_m);
  memset(g2, 0, sizeof(double) * NG2 * (size_t)n);
  memset(m2, 0, sizeof(double) * NG2 * (size_t)n);
  for (int64_t p = 0; p < P; ++p) { /* fixed (tile, depth) order: deterministic */
    int g = sorted_idx[p];
    for (int j = 0; j < NG2; ++j) {
      g2[(size_t)g * NG2 + j] += pair_g[(size_t)p * NG2 + j];
      m2[(size_t)g * NG2 + j] += pair_m[(size_t)p * NG2 + j];
    }
  }
  free(pair_g);
  free(pair_m);
  int nthr = 1;
#ifdef _OPENMP
  nthr = omp_get_max_threads();
#endif
  double *pacc = (double *)calloc((size_t)nthr * 24, sizeof(double));
#pragma omp parallel
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
#pragma omp for schedule(static)
    for (int i = 0; i < n; ++i) {
      ogauss G;
      project_one(mean + 3 * i, quat + 4 * i, logscale + 3 * i, logit[i], R, t, &k, &G);
      double *o3 = g3 + (size_t)i * 16, *om = m3 + (size_t)i * 16;
      if (G.culled) {
        memset(o3, 0, sizeof(double) * 16);
        memset(om, 0, sizeof(double) * 16);
        continue;
      }
      double pp[12];
      chain3d(&G, mean + 3 * i, R, &k, g2 + (size_t)i * NG2, o3, pp);
      /* magnitude: |J^T| m2 via the 10 unit columns of the (linear) chain */
      double e[NG2], col3[16], colp[12], mp[12];
      memset(om, 0, sizeof(double) * 16);
      memset(mp, 0, sizeof(mp));
      for (int j = 0; j < NG2; ++j) {
        double mj = m2[(size_t)i * NG2 + j];
        if (mj == 0.0) continue;
        memset(e, 0, sizeof(e));
        e[j] = 1.0;
        chain3d(&G, mean + 3 * i, R, &k, e, col3, colp);
        for (int c = 0; c < 16; ++c) om[c] += fabs(col3[c]) * mj;
        for (int c = 0; c < 12; ++c) mp[c] += fabs(colp[c]) * mj;
      }
      for (int c = 0; c < 12; ++c) {
        pacc[tid * 24 + c] += pp[c];
        pacc[tid * 24 + 12 + c] += mp[c];
      }
    }
  }
  if (pose) memset(pose, 0, sizeof(double) * 12);
  if (mpose) memset(mpose, 0, sizeof(double) * 12);
  for (int th = 0; th < nthr; ++th)
    for (int c = 0; c < 12; ++c) {
      if (pose) pose[c] += pacc[th * 24 + c];
      if (mpose) mpose[c] += pacc[th * 24 + 12 + c];
    }
  free(pacc);
  free(uv);
  free(conic);
  free(opac);
  free(pz);
}

/* ------------------------------------------------------------------ */
/* S7 pose gradient conversions (Eq. 14; R22).                 */

/* Left-perturbation twist xi = (v, w), T <- exp(xi^) T:
 *   R' = exp(w^) R, t' = exp(w^) t + v (first order)
 *   dL/dv = dL/dt;  dL/dw_k = <dL/dR, [e_k]x R> + dL/dt . (e_k x t). */
void or_pose_twist(const double *gR, const double *gt, const double *R, const double *t,
                   double *twist) {
  for (int i = 0; i < 3; ++i) twist[i] = gt[i];
  for (int kk = 0; kk < 3; ++kk) {
    double E[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}; /* [e_k]x */
    double e[3] = {0, 0, 0};
    e[kk] = 1.0;
    E[1] = -e[2]; E[2] = e[1];
    E[3] = e[2];  E[5] = -e[0];
    E[6] = -e[1]; E[7] = e[0];
    double acc = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double ER = 0.0;
        for (int c = 0; c < 3; ++c) ER += E[3 * a + c] * R[3 * c + b];
        acc += gR[3 * a + b] * ER;
      }
    double ext[3] = {e[1] * t[2] - e[2] * t[1], e[2] * t[0] - e[0] * t[2], e[0] * t[1] - e[1] * t[0]};
    acc += gt[0] * ext[0] + gt[1] * ext[1] + gt[2] * ext[2];
    twist[3 + kk] = acc;
  }
}

/* (q, t) parameterisation: R = R(q^), q unit (w, x, y, z).
 * dL/dq = (I - q q^T) sum_ij dL/dR_ij dR_ij/dq. */
void or_pose_qt(const double *gR, const double *q, double *gq) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double dw[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
  double dx[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
  double dy[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
  double dz[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
  double g[4] = {0, 0, 0, 0};
  for (int i = 0; i < 9; ++i) {
    g[0] += gR[i] * dw[i];
    g[1] += gR[i] * dx[i];
    g[2] += gR[i] * dy[i];
    g[3] += gR[i] * dz[i];
  }
  double dot = g[0] * w + g[1] * x + g[2] * y + g[3] * z;
  for (int i = 0; i < 4; ++i) gq[i] = g[i] - q[i] * dot;
}

/* SO(3)/SE(3) exponential (Rodrigues + left Jacobian V) of xi = (v, w). */
void or_se3_exp(const double *xi, double *R, double *t) {
  const double *v = xi, *w = xi + 3;
  double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2], th = sqrt(th2);
  double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0}, K2[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += K[3 * a + c] * K[3 * c + b];
      K2[3 * a + b] = acc;
    }
  double A, B, Cc;
  if (th < 1e-8) {
    A = 1.0 - th2 / 6.0;
    B = 0.5 - th2 / 24.0;
    Cc = 1.0 / 6.0 - th2 / 120.0;
  } else {
    A = sin(th) / th;
    B = (1.0 - cos(th)) / th2;
    Cc = (th - sin(th)) / (th2 * th);
  }
  double V[9];
  for (int i = 0; i < 9; ++i) {
    double I = (i % 4 == 0) ? 1.0 : 0.0;
    R[i] = I + A * K[i] + B * K2[i];
    V[i] = I + B * K[i] + Cc * K2[i];
  }
  for (int i = 0; i < 3; ++i) t[i] = V[3 * i] * v[0] + V[3 * i + 1] * v[1] + V[3 * i + 2] * v[2];
}

/* One Adam step on the twist, applied as T <- exp(-d^) T with
 * d_i = lr_i mhat_i / (sqrt(vhat_i) + eps).  state[13] = m[6], v[6], step.
 * lr[2] = (lr_trans, lr_rot); hyp[3] = (beta1, beta2, eps). */
void or_pose_adam(double *R, double *t, const double *twist_grad, double *state,
                  const double *lr, const double *hyp) {
  double b1 = hyp[0], b2 = hyp[1], eps = hyp[2];
  state[12] += 1.0;
  double stp = state[12];
  double d[6];
  for (int i = 0; i < 6; ++i) {
    state[i] = b1 * state[i] + (1.0 - b1) * twist_grad[i];
    state[6 + i] = b2 * state[6 + i] + (1.0 - b2) * twist_grad[i] * twist_grad[i];
    double mh = state[i] / (1.0 - pow(b1, stp));
    double vh = state[6 + i] / (1.0 - pow(b2, stp));
    d[i] = -(i < 3 ? lr[0] : lr[1]) * mh / (sqrt(vh) + eps);
  }
  double dR[9], dt[3], R2[9], t2[3];
  or_se3_exp(d, dR, dt);
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 3; ++c) acc += dR[3 * a + c] * R[3 * c + b];
      R2[3 * a + b] = acc;
    }
    t2[a] = dR[3 * a] * t[0] + dR[3 * a + 1] * t[1] + dR[3 * a + 2] * t[2] + dt[a];
  }
  memcpy(R, R2, sizeof(R2));
  memcpy(t, t2, sizeof(t2));
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
