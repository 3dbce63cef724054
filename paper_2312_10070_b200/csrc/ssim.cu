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
// Two separable passes, each one CTA per (16x16 tile, channel) with a 26x26
// halo in shared memory: k_ssim_stats (the five local moments -> S, A, B, Cc)
// and k_ssim_grad (the three blurred maps -> the gradient, added to
// dL_dcolor); fp64 block partials of S, reduced in a fixed order.
#include <cmath>

#include "gs_internal.cuh"

namespace gs {

constexpr int kSR = 5;                 // window radius
constexpr int kSW = 2 * kSR + 1;       // 11 taps
constexpr int kSH = kTile + 2 * kSR;   // 26: halo tile side
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

struct SsimTaps {
  float g[kSW];
};

struct SsimArgs {
  const float *x, *y;  // rendered [3][H][W], target [3][H][W]
  int W, H, TX;
  float *A, *B, *Cc;   // [3][H][W] each
  double *part;        // [3 * tiles]
  float weight;        // dL_dcolor += -weight * dSSIM/dx
  float *g_color, *loss;
};

// Zero-padded halo tile of a [H][W] map around tile (tx, ty), in-image
// values shifted by `shift`.
__device__ __forceinline__ void load_halo(float (*s)[kSH], const float *m, int tx, int ty, int W, int H,
                                          float shift = 0.f) {
  for (int i = threadIdx.x; i < kSH * kSH; i += blockDim.x) {
    const int r = i / kSH, c = i % kSH;
    const int gy = ty * kTile - kSR + r, gx = tx * kTile - kSR + c;
    s[r][c] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? __ldg(m + size_t(gy) * W + gx) - shift : 0.f;
  }
}

// Window mass inside the image at coordinate p of an axis of length n.
__device__ __forceinline__ float axis_mass(const SsimTaps &t, int p, int n) {
  float m = 0.f;
#pragma unroll
  for (int k = 0; k < kSW; ++k) m += (p + k - kSR >= 0 && p + k - kSR < n) ? t.g[k] : 0.f;
  return m;
}

__global__ void __launch_bounds__(256) k_ssim_stats(SsimArgs a, SsimTaps t) {
  __shared__ float sx[kSH][kSH], sy[kSH][kSH];
  __shared__ float h[5][kSH][kTile];
  __shared__ double sh[256];
  const int tx = blockIdx.x % a.TX, ty = blockIdx.x / a.TX, ch = blockIdx.y;
  const size_t HW = size_t(a.W) * a.H;
  // moments of the in-image values shifted by the tile's first pixel (cx, cy):
  // the variances / covariance then carry no cancellation of the squared
  // means (exact zeros on flat patches); the mass m = G*1_image restores the
  // zero-padded statistics exactly (see below)
  const size_t o = ch * HW + size_t(ty * kTile) * a.W + tx * kTile;
  const float cx = __ldg(a.x + o), cy = __ldg(a.y + o);
  load_halo(sx, a.x + ch * HW, tx, ty, a.W, a.H, cx);
  load_halo(sy, a.y + ch * HW, tx, ty, a.W, a.H, cy);
  __syncthreads();
  // horizontal pass: the five moments over 26 rows x 16 columns
  for (int i = threadIdx.x; i < kSH * kTile; i += blockDim.x) {
    const int r = i / kTile, c = i % kTile;
    float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
    for (int k = 0; k < kSW; ++k) {
      const float xv = sx[r][c + k], yv = sy[r][c + k], g = t.g[k];
      m0 = fmaf(g, xv, m0);
      m1 = fmaf(g, yv, m1);
      m2 = fmaf(g, xv * xv, m2);
      m3 = fmaf(g, yv * yv, m3);
      m4 = fmaf(g, xv * yv, m4);
    }
    h[0][r][c] = m0;
    h[1][r][c] = m1;
    h[2][r][c] = m2;
    h[3][r][c] = m3;
    h[4][r][c] = m4;
  }
  __syncthreads();
  const int i = threadIdx.x / kTile, j = threadIdx.x % kTile;
  float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < kSW; ++k) {
    const float g = t.g[k];
#pragma unroll
    for (int q = 0; q < 5; ++q) m[q] = fmaf(g, h[q][i + k][j], m[q]);
  }
  const int px = tx * kTile + j, py = ty * kTile + i;
  double s_acc = 0.0;
  if (px < a.W && py < a.H) {
    // shifted moments G1 = G*x', G2 = G*y' with x' = (x - cx) 1_image:
    //   mu_x = G1 + cx m,  s_xx = G*x'^2 - G1^2 + (2 cx G1 + cx^2 m)(1 - m),
    //   s_xy = G*x'y' - G1 G2 + (cx G2 + cy G1 + cx cy m)(1 - m)
    const float mass = axis_mass(t, px, a.W) * axis_mass(t, py, a.H), om = 1.f - mass;
    const float G1 = m[0], G2 = m[1];
    const float mx = fmaf(cx, mass, G1), my = fmaf(cy, mass, G2);
    const float sxx = (m[2] - G1 * G1) + (2.f * cx * G1 + cx * cx * mass) * om;
    const float syy = (m[3] - G2 * G2) + (2.f * cy * G2 + cy * cy * mass) * om;
    const float sxy = (m[4] - G1 * G2) + (cx * G2 + cy * G1 + cx * cy * mass) * om;
    const float n1 = 2.f * mx * my + kC1, n2 = 2.f * sxy + kC2;
    const float d1 = mx * mx + my * my + kC1, d2 = sxx + syy + kC2;
    const float D = d1 * d2, iD = 1.f / D;
    const float S = n1 * n2 * iD;
    const float dmx = 2.f * my * n2 * iD - 2.f * mx * S / d1;
    const float dsxx = -S / d2, dsxy = 2.f * n1 * iD;
    const size_t q = ch * HW + size_t(py) * a.W + px;
    a.A[q] = dmx - 2.f * mx * dsxx - my * dsxy;
    a.B[q] = dsxx;
    a.Cc[q] = dsxy;
    s_acc = double(S);
  }
  // fixed-shape block tree: deterministic
  sh[threadIdx.x] = s_acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.part[blockIdx.y * gridDim.x + blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) k_ssim_grad(SsimArgs a, SsimTaps t) {
  __shared__ float sm[3][kSH][kSH];
  __shared__ float h[3][kSH][kTile];
  const int tx = blockIdx.x % a.TX, ty = blockIdx.x / a.TX, ch = blockIdx.y;
  const size_t HW = size_t(a.W) * a.H;
  load_halo(sm[0], a.A + ch * HW, tx, ty, a.W, a.H);
  load_halo(sm[1], a.B + ch * HW, tx, ty, a.W, a.H);
  load_halo(sm[2], a.Cc + ch * HW, tx, ty, a.W, a.H);
  __syncthreads();
  for (int i = threadIdx.x; i < kSH * kTile; i += blockDim.x) {
    const int r = i / kTile, c = i % kTile;
    float m0 = 0.f, m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int k = 0; k < kSW; ++k) {
      const float g = t.g[k];
      m0 = fmaf(g, sm[0][r][c + k], m0);
      m1 = fmaf(g, sm[1][r][c + k], m1);
      m2 = fmaf(g, sm[2][r][c + k], m2);
    }
    h[0][r][c] = m0;
    h[1][r][c] = m1;
    h[2][r][c] = m2;
  }
  __syncthreads();
  const int i = threadIdx.x / kTile, j = threadIdx.x % kTile;
  const int px = tx * kTile + j, py = ty * kTile + i;
  if (px >= a.W || py >= a.H) return;
  float bA = 0.f, bB = 0.f, bC = 0.f;
#pragma unroll
  for (int k = 0; k < kSW; ++k) {
    const float g = t.g[k];
    bA = fmaf(g, h[0][i + k][j], bA);
    bB = fmaf(g, h[1][i + k][j], bB);
    bC = fmaf(g, h[2][i + k][j], bC);
  }
  const size_t q = ch * HW + size_t(py) * a.W + px;
  const float xv = __ldg(a.x + q), yv = __ldg(a.y + q);
  const float grad = bA + 2.f * xv * bB + yv * bC;  // 3HW x dSSIM/dx
  a.g_color[q] += -a.weight / float(3 * HW) * grad;
}

__global__ void __launch_bounds__(256) k_ssim_final(SsimArgs a, int nblk) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += a.part[b];  // fixed order per thread
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double ssim = sh[0] / (3.0 * double(a.W) * double(a.H));
    a.loss[0] += float(double(a.weight) * (1.0 - ssim));
    a.loss[3] = float(ssim);
  }
}

static size_t ssim_ws_bytes(const gs_camera &cam) {
  const size_t HW = size_t(cam.width) * cam.height;
  const size_t nblk = size_t(3) * tiles_x(cam) * tiles_y(cam);
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
  const int T = tiles_x(cam) * tiles_y(cam);
  SsimArgs a{color, tgt_color, cam.width, cam.height, tiles_x(cam), A, A + 3 * HW, A + 6 * HW,
             reinterpret_cast<double *>(A + 9 * HW + (9 * HW & 1)), weight, dL_dcolor, loss};
  SsimTaps t;
  double g[kSW], sum = 0.0;
  for (int k = 0; k < kSW; ++k) {
    g[k] = std::exp(-double((k - kSR) * (k - kSR)) / (2.0 * 1.5 * 1.5));
    sum += g[k];
  }
  for (int k = 0; k < kSW; ++k) t.g[k] = float(g[k] / sum);
  cudaStream_t s = as_stream(stream);
  const dim3 grid(T, 3);
  k_ssim_stats<<<grid, 256, 0, s>>>(a, t);
  k_ssim_grad<<<grid, 256, 0, s>>>(a, t);
  k_ssim_final<<<1, 256, 0, s>>>(a, 3 * T);
  return check_launch("gs_ssim");
}
