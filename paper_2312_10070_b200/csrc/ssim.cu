// ssim.cu — NEXT(2) gs_ssim: the SSIM term of the colour loss (Eq. 10,
// P:184-190; R32-R33).
//
// Per channel and pixel p (Wang et al. 2004, the paper's [wang2004image]):
//   mu_x = G*x, mu_y = G*y, s_xx = G*(x^2) - mu_x^2, s_yy = G*(y^2) - mu_y^2,
//   s_xy = G*(xy) - mu_x mu_y,
//   S(p) = (2 mu_x mu_y + C1)(2 s_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(s_xx + s_yy + C2)),
// G the 11x11 Gaussian window (sigma 1.5) applied as a zero-padded "same"
// correlation; SSIM = mean of S over 3HW.  Its gradient w.r.t. the rendered
// image x (y = target):
//   dSSIM/dx(q) = [G*A + 2 x G*B + y G*Cc](q) / 3HW,
//   A = dS/dmu_x - 2 mu_x dS/ds_xx - mu_y dS/ds_xy, B = dS/ds_xx, Cc = dS/ds_xy.
// Two separable passes, each one CTA per (32x32 tile, channel) with a 42x42
// halo in shared memory, the window sliding over register-held rows (8
// outputs per horizontal task, 4 per vertical one): k_ssim_stats (the five
// local moments -> S, A, B, Cc) and k_ssim_grad (the three blurred maps ->
// the gradient, added to dL_dcolor); fp64 block partials of S, reduced in a
// fixed order.
#include <cmath>

#include "gs_internal.cuh"

namespace gs {

constexpr int kSR = 5;                  // window radius
constexpr int kSW = 2 * kSR + 1;        // 11 taps
constexpr int kST = 32;                 // output tile side (32 x 32 per CTA)
constexpr int kSH = kST + 2 * kSR;      // 42: halo tile side
constexpr int kSThreads = 256;
constexpr int kHSeg = 8;                // horizontal pass: 8 outputs per thread task (sliding window)
constexpr int kVSeg = 4;                // vertical pass: 4 outputs per thread
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

struct SsimTaps {
  float g[kSW];
};

struct SsimArgs {
  const float *x, *y;  // rendered [3][H][W], target [3][H][W]
  int W, H, TX;        // TX = tiles of kST columns
  float *A, *B, *Cc;   // [3][H][W] each
  double *part;        // [3 * tiles]
  float weight;        // dL_dcolor += -weight * dSSIM/dx
  float *g_color, *loss;
};

// Zero-padded kSH x kSH halo of a [H][W] map around output tile (tx, ty),
// in-image values shifted by `shift`.
__device__ __forceinline__ void load_halo(float (*s)[kSH], const float *m, int tx, int ty, int W, int H,
                                          float shift = 0.f) {
  // 64 threads per row (42 used), 4 rows per pass: all 11 loads of a thread
  // are issued before the first store (latency-bound otherwise)
  constexpr int kRowsPer = (kSH + kSThreads / 64 - 1) / (kSThreads / 64);  // 11
  const int gy0 = ty * kST - kSR, gx0 = tx * kST - kSR;
  const int c = threadIdx.x % 64, r0 = threadIdx.x / 64;
  const int gx = gx0 + c;
  const bool colin = c < kSH && gx >= 0 && gx < W;
  float v[kRowsPer];
#pragma unroll
  for (int i = 0; i < kRowsPer; ++i) {
    const int r = r0 + i * (kSThreads / 64), gy = gy0 + r;
    v[i] = (colin && r < kSH && gy >= 0 && gy < H) ? __ldg(m + size_t(gy) * W + gx) - shift : 0.f;
  }
  if (c < kSH) {
#pragma unroll
    for (int i = 0; i < kRowsPer; ++i) {
      const int r = r0 + i * (kSThreads / 64);
      if (r < kSH) s[r][c] = v[i];
    }
  }
}

// Window mass inside the image at coordinate p of an axis of length n.
__device__ __forceinline__ float axis_mass(const SsimTaps &t, int p, int n) {
  float m = 0.f;
#pragma unroll
  for (int k = 0; k < kSW; ++k) m += (p + k - kSR >= 0 && p + k - kSR < n) ? t.g[k] : 0.f;
  return m;
}

// Horizontal pass of NM maps over the halo: out[q][r][c] = sum_k g_k in_q(r, c + k)
// for r < kSH, c < kST.  A task = one row and kHSeg consecutive outputs: the
// kHSeg + 10 inputs are read once into registers and the window slides.
template <int NM, class F>
__device__ __forceinline__ void hpass(const SsimTaps &t, F in, float (*out)[kSH][kST]) {
  constexpr int kTasks = kSH * (kST / kHSeg);  // 168
  for (int task = threadIdx.x; task < kTasks; task += kSThreads) {
    const int r = task / (kST / kHSeg), c0 = (task % (kST / kHSeg)) * kHSeg;
    float v[NM][kHSeg + 2 * kSR];
#pragma unroll
    for (int k = 0; k < kHSeg + 2 * kSR; ++k) in(r, c0 + k, v, k);
#pragma unroll
    for (int o = 0; o < kHSeg; ++o) {
      float acc[NM];
#pragma unroll
      for (int q = 0; q < NM; ++q) acc[q] = 0.f;
#pragma unroll
      for (int k = 0; k < kSW; ++k)
#pragma unroll
        for (int q = 0; q < NM; ++q) acc[q] = fmaf(t.g[k], v[q][o + k], acc[q]);
#pragma unroll
      for (int q = 0; q < NM; ++q) out[q][r][c0 + o] = acc[q];
    }
  }
}

// Vertical pass for this thread's kVSeg outputs of column c, rows r0..r0+3.
template <int NM>
__device__ __forceinline__ void vpass(const SsimTaps &t, const float (*h)[kSH][kST], int r0, int c,
                                      float res[kVSeg][NM]) {
#pragma unroll
  for (int o = 0; o < kVSeg; ++o)
#pragma unroll
    for (int q = 0; q < NM; ++q) res[o][q] = 0.f;
#pragma unroll
  for (int k = 0; k < kVSeg + 2 * kSR; ++k) {
#pragma unroll
    for (int q = 0; q < NM; ++q) {
      const float v = h[q][r0 + k][c];
#pragma unroll
      for (int o = 0; o < kVSeg; ++o)
        if (k - o >= 0 && k - o < kSW) res[o][q] = fmaf(t.g[k - o], v, res[o][q]);
    }
  }
}

struct StatsSmem {
  float sx[kSH][kSH], sy[kSH][kSH];
  float h[5][kSH][kST];
  double red[kSThreads / 32];
};

__global__ void __launch_bounds__(kSThreads) k_ssim_stats(SsimArgs a, SsimTaps t) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StatsSmem &S = *reinterpret_cast<StatsSmem *>(smem_raw);
  const int tx = blockIdx.x % a.TX, ty = blockIdx.x / a.TX, ch = blockIdx.y;
  const size_t HW = size_t(a.W) * a.H;
  // moments of the in-image values shifted by the tile's first pixel (cx, cy):
  // the variances / covariance then carry no cancellation of the squared
  // means (exact zeros on flat patches); the mass m = G*1_image restores the
  // zero-padded statistics exactly (see below)
  const size_t o0 = ch * HW + size_t(ty * kST) * a.W + tx * kST;
  const float cx = __ldg(a.x + o0), cy = __ldg(a.y + o0);
  load_halo(S.sx, a.x + ch * HW, tx, ty, a.W, a.H, cx);
  load_halo(S.sy, a.y + ch * HW, tx, ty, a.W, a.H, cy);
  __syncthreads();
  hpass<5>(t, [&](int r, int c, float (*v)[kHSeg + 2 * kSR], int k) {
    const float xv = S.sx[r][c], yv = S.sy[r][c];
    v[0][k] = xv;
    v[1][k] = yv;
    v[2][k] = xv * xv;
    v[3][k] = yv * yv;
    v[4][k] = xv * yv;
  }, S.h);
  __syncthreads();
  const int c = threadIdx.x % kST, r0 = (threadIdx.x / kST) * kVSeg;
  float m[kVSeg][5];
  vpass<5>(t, S.h, r0, c, m);
  double s_acc = 0.0;
  const int px = tx * kST + c;
  const float massx = axis_mass(t, px, a.W);
#pragma unroll
  for (int o = 0; o < kVSeg; ++o) {
    const int py = ty * kST + r0 + o;
    if (px >= a.W || py >= a.H) continue;
    // shifted moments G1 = G*x', G2 = G*y' with x' = (x - cx) 1_image:
    //   mu_x = G1 + cx m,  s_xx = G*x'^2 - G1^2 + (2 cx G1 + cx^2 m)(1 - m),
    //   s_xy = G*x'y' - G1 G2 + (cx G2 + cy G1 + cx cy m)(1 - m)
    const float mass = massx * axis_mass(t, py, a.H), om = 1.f - mass;
    const float G1 = m[o][0], G2 = m[o][1];
    const float mx = fmaf(cx, mass, G1), my = fmaf(cy, mass, G2);
    const float sxx = (m[o][2] - G1 * G1) + (2.f * cx * G1 + cx * cx * mass) * om;
    const float syy = (m[o][3] - G2 * G2) + (2.f * cy * G2 + cy * cy * mass) * om;
    const float sxy = (m[o][4] - G1 * G2) + (cx * G2 + cy * G1 + cx * cy * mass) * om;
    const float n1 = 2.f * mx * my + kC1, n2 = 2.f * sxy + kC2;
    const float d1 = mx * mx + my * my + kC1, d2 = sxx + syy + kC2;
    const float iD = 1.f / (d1 * d2);
    const float Sv = n1 * n2 * iD;
    const float dmx = 2.f * my * n2 * iD - 2.f * mx * Sv / d1;
    const float dsxx = -Sv / d2, dsxy = 2.f * n1 * iD;
    const size_t q = ch * HW + size_t(py) * a.W + px;
    a.A[q] = dmx - 2.f * mx * dsxx - my * dsxy;
    a.B[q] = dsxx;
    a.Cc[q] = dsxy;
    s_acc += double(Sv);
  }
  // fixed-order block sum: warp tree, then the 8 warp sums in order
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s_acc += __shfl_xor_sync(0xffffffffu, s_acc, off);
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5] = s_acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < kSThreads / 32; ++w) b += S.red[w];
    a.part[blockIdx.y * gridDim.x + blockIdx.x] = b;
  }
}

struct GradSmem {
  float sm[3][kSH][kSH];
  float h[3][kSH][kST];
};

__global__ void __launch_bounds__(kSThreads) k_ssim_grad(SsimArgs a, SsimTaps t) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GradSmem &S = *reinterpret_cast<GradSmem *>(smem_raw);
  const int tx = blockIdx.x % a.TX, ty = blockIdx.x / a.TX, ch = blockIdx.y;
  const size_t HW = size_t(a.W) * a.H;
  load_halo(S.sm[0], a.A + ch * HW, tx, ty, a.W, a.H);
  load_halo(S.sm[1], a.B + ch * HW, tx, ty, a.W, a.H);
  load_halo(S.sm[2], a.Cc + ch * HW, tx, ty, a.W, a.H);
  __syncthreads();
  hpass<3>(t, [&](int r, int c, float (*v)[kHSeg + 2 * kSR], int k) {
    v[0][k] = S.sm[0][r][c];
    v[1][k] = S.sm[1][r][c];
    v[2][k] = S.sm[2][r][c];
  }, S.h);
  __syncthreads();
  const int c = threadIdx.x % kST, r0 = (threadIdx.x / kST) * kVSeg;
  float m[kVSeg][3];
  vpass<3>(t, S.h, r0, c, m);
  const int px = tx * kST + c;
  const float sc = -a.weight / float(3 * HW);
#pragma unroll
  for (int o = 0; o < kVSeg; ++o) {
    const int py = ty * kST + r0 + o;
    if (px >= a.W || py >= a.H) continue;
    const size_t q = ch * HW + size_t(py) * a.W + px;
    const float xv = __ldg(a.x + q), yv = __ldg(a.y + q);
    const float grad = m[o][0] + 2.f * xv * m[o][1] + yv * m[o][2];  // 3HW x dSSIM/dx
    a.g_color[q] += sc * grad;
  }
}

__global__ void __launch_bounds__(1024) k_ssim_final(SsimArgs a, int nblk) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += a.part[b];  // fixed order per thread
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = 512; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double ssim = sh[0] / (3.0 * double(a.W) * double(a.H));
    a.loss[0] += float(double(a.weight) * (1.0 - ssim));
    a.loss[3] = float(ssim);
  }
}

static int ssim_tiles_x(const gs_camera &c) { return (c.width + kST - 1) / kST; }
static int ssim_tiles_y(const gs_camera &c) { return (c.height + kST - 1) / kST; }

static size_t ssim_ws_bytes(const gs_camera &cam) {
  const size_t HW = size_t(cam.width) * cam.height;
  const size_t nblk = size_t(3) * ssim_tiles_x(cam) * ssim_tiles_y(cam);
  return 3 * 3 * HW * sizeof(float) + nblk * sizeof(double) + 256;
}

}  // namespace gs

extern "C" size_t gs_ssim_workspace_bytes(gs_camera cam) {
  if (!gs::camera_ok(cam)) return 0;
  return gs::ssim_ws_bytes(cam);
}

extern "C" int gs_ssim(gs_camera cam, const float *color, const float *tgt_color, float weight, void *ws,
                       size_t ws_bytes, float *loss, float *dL_dcolor, void *stream) {
  using namespace gs;
  if (!camera_ok(cam) || !color || !tgt_color || !loss || !dL_dcolor || !(weight >= 0.f)) {
    set_error("gs_ssim: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (!ws || ws_bytes < ssim_ws_bytes(cam)) {
    set_error("gs_ssim: workspace %zu < %zu bytes", ws_bytes, ssim_ws_bytes(cam));
    return GS_ERR_WORKSPACE;
  }
  const size_t HW = size_t(cam.width) * cam.height;
  float *A = static_cast<float *>(ws);
  const int T = ssim_tiles_x(cam) * ssim_tiles_y(cam);
  SsimArgs a{color, tgt_color, cam.width, cam.height, ssim_tiles_x(cam), A, A + 3 * HW, A + 6 * HW,
             reinterpret_cast<double *>(A + 9 * HW + (9 * HW & 1)), weight, dL_dcolor, loss};
  SsimTaps t;
  double g[kSW], sum = 0.0;
  for (int k = 0; k < kSW; ++k) {
    g[k] = std::exp(-double((k - kSR) * (k - kSR)) / (2.0 * 1.5 * 1.5));
    sum += g[k];
  }
  for (int k = 0; k < kSW; ++k) t.g[k] = float(g[k] / sum);
  cudaStream_t s = as_stream(stream);
  static thread_local bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ssim_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(StatsSmem)));
    cudaFuncSetAttribute(k_ssim_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(GradSmem)));
    attr = true;
  }
  const dim3 grid(T, 3);
  k_ssim_stats<<<grid, kSThreads, sizeof(StatsSmem), s>>>(a, t);
  k_ssim_grad<<<grid, kSThreads, sizeof(GradSmem), s>>>(a, t);
  k_ssim_final<<<1, 1024, 0, s>>>(a, 3 * T);
  return check_launch("gs_ssim");
}
