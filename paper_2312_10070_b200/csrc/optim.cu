// optim.cu — NEXT(3): the device epilogue of a mapping iteration.
//
//  * gs_iso_reg: the isotropic regulariser of Eq. 11,
//      L_reg = sum_k |s_k - s^bar_k|_1 / |K|,  s_k = exp(logscale_k) in R^3,
//      s^bar_k = the mean of s_k's three components (R34),
//    added (x lambda_reg, Eq. 12) to loss[0] and its gradient to the
//    log-scale gradients (chain through exp).
//  * gs_adam_step: one Adam step (bias-corrected moments, per-group
//    learning rates, quaternions renormalised after the step, Gaussians with
//    a non-finite gradient skipped and counted) over the float4 SoA parameters,
//    in place; the moments live in one [n][8] float4 buffer (m of the four
//    arrays, then v), so pruning compacts them with the parameters.
//  * gs_prune: removes the Gaussians whose opacity sigmoid(logit) < o_thre
//    (P:624), a stable compaction of the parameters and the Adam moments.
// All per-Gaussian kernels are coalesced float4 passes (HBM-bound); the
// regulariser's sum and the prune scan are fixed-order (deterministic).
#include <algorithm>
#include <cmath>

#include "gs_internal.cuh"

namespace gs {

constexpr int kOptThreads = 256;

__device__ __forceinline__ float sgnf(float x) { return float((x > 0.f) - (x < 0.f)); }

// ---- Eq. 11 ------------------------------------------------------------------
__global__ void __launch_bounds__(kOptThreads) k_iso_reg(const float4 *__restrict__ logscale, int n, float w,
                                                         float4 *g_logscale, double *part) {
  __shared__ double sh[kOptThreads / 32];
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float4 l = __ldg(logscale + i);
    const float s0 = expf(l.x), s1 = expf(l.y), s2 = expf(l.z);
    const float sb = (s0 + s1 + s2) * (1.f / 3.f);
    const float d0 = sgnf(s0 - sb), d1 = sgnf(s1 - sb), d2 = sgnf(s2 - sb);
    acc += double(fabsf(s0 - sb)) + double(fabsf(s1 - sb)) + double(fabsf(s2 - sb));
    // dL/ds_j = (sign_j - mean(sign)) / |K|; dL/dlogscale_j = dL/ds_j s_j
    const float dm = (d0 + d1 + d2) * (1.f / 3.f);
    float4 g = g_logscale[i];
    g.x += w * (d0 - dm) * s0;
    g.y += w * (d1 - dm) * s1;
    g.z += w * (d2 - dm) * s2;
    g_logscale[i] = g;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int k = 0; k < kOptThreads / 32; ++k) b += sh[k];
    part[blockIdx.x] = b;
  }
}

__global__ void __launch_bounds__(kOptThreads) k_iso_reg_final(const double *part, int nblk, int n, float lambda,
                                                               float *loss) {
  __shared__ double sh[kOptThreads];
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += part[b];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = kOptThreads / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0 && n > 0) {
    const double reg = sh[0] / double(n);
    loss[0] += float(double(lambda) * reg);
    loss[1] = float(reg);
  }
}

// ---- Adam ----------------------------------------------------------------------
struct AdamArgs {
  float4 *p[4];        // mean_opa, quat, logscale, rgb (in place)
  const float4 *g[4];  // gradients, same layout
  float4 *mv;          // [n][8]: m[4], v[4]
  int n;
  float lr[4][4];      // per array and component
  float b1, b2, omb1, omb2, eps, c1, c2;  // omb = 1 - b (from fp64: no fp32 cancellation), c = 1 - b^t
  gs_counters *cnt;
};

__device__ __forceinline__ bool finite4(float4 a) {
  return isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w);
}

__global__ void __launch_bounds__(kOptThreads) k_adam(AdamArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool skipped = false;
  if (i < a.n) {
    float4 g[4];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      g[k] = __ldg(a.g[k] + i);
      ok &= finite4(g[k]);
    }
    if (!ok) {
      skipped = true;  // skip the entry, count it
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float4 *mq = a.mv + size_t(i) * 8 + k, *vq = mq + 4;
        float4 m = *mq, v = *vq, p = a.p[k][i];
        float *pm = &m.x, *pv = &v.x, *pp = &p.x;
        const float *pg = &g[k].x;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          pm[c] = a.b1 * pm[c] + a.omb1 * pg[c];
          pv[c] = a.b2 * pv[c] + a.omb2 * pg[c] * pg[c];
          const float mh = pm[c] / a.c1, vh = pv[c] / a.c2;
          pp[c] -= a.lr[k][c] * mh / (sqrtf(vh) + a.eps);
        }
        if (k == 1) {  // quaternions renormalised after the step
          const float r = rsqrtf(p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w);
          p = make_float4(p.x * r, p.y * r, p.z * r, p.w * r);
        }
        *mq = m;
        *vq = v;
        a.p[k][i] = p;
      }
    }
  }
  if (a.cnt) {
    const unsigned ns = __popc(__ballot_sync(0xffffffffu, skipped));
    if ((threadIdx.x & 31) == 0) count_add(&a.cnt->n_nonfinite, ns);
  }
}

// ---- pruning: stable compaction -------------------------------------------------
// prune when the opacity sigmoid(logit) < o_thre; decided in fp64
// (R35)
__device__ __forceinline__ bool keep_gauss(const float4 *mo, int i, double o_thre) {
  return 1.0 / (1.0 + exp(-double(__ldg(mo + i).w))) >= o_thre;
}

__global__ void __launch_bounds__(kOptThreads) k_prune_count(const float4 *mo, int n, double lt, int *bcount) {
  __shared__ int sh[kOptThreads / 32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool k = i < n && keep_gauss(mo, i, lt);
  const int c = __popc(__ballot_sync(0xffffffffu, k));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kOptThreads / 32; ++w) s += sh[w];
    bcount[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(1024) k_prune_scan(int *bcount, int nblk, int *n_out) {
  // exclusive scan of the block counts in place (one CTA, sequential chunks)
  __shared__ int sh[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblk; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const int v = b < nblk ? bcount[b] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int y = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += y;
      __syncthreads();
    }
    if (b < nblk) bcount[b] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = carry;
}

struct PruneArgs {
  const float4 *src[4], *ms;  // params, moments [n][8] (nullable)
  float4 *dst[4], *md;
  int n;
  double lt;
  const int *boff;
};

__global__ void __launch_bounds__(kOptThreads) k_prune_scatter(PruneArgs a) {
  __shared__ int sh[kOptThreads / 32];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool k = i < a.n && keep_gauss(a.src[0], i, a.lt);
  const unsigned b = __ballot_sync(0xffffffffu, k);
  if (lane == 0) sh[w] = __popc(b);
  __syncthreads();
  int before = a.boff[blockIdx.x];
  for (int ww = 0; ww < w; ++ww) before += sh[ww];
  if (!k) return;
  const int o = before + __popc(b & lanemask_lt());
#pragma unroll
  for (int q = 0; q < 4; ++q) a.dst[q][o] = __ldg(a.src[q] + i);
  if (a.ms) {
#pragma unroll
    for (int q = 0; q < 8; ++q) a.md[size_t(o) * 8 + q] = a.ms[size_t(i) * 8 + q];
  }
}

}  // namespace gs

extern "C" size_t gs_opt_workspace_bytes(int32_t n) {
  return size_t(8) * (size_t((n + gs::kOptThreads - 1) / gs::kOptThreads) + 1) + 256;
}

extern "C" int gs_iso_reg(gs_params p, float lambda_reg, float *g_logscale_, void *ws, size_t ws_bytes,
                          float *loss, void *stream) {
  float4 *g_logscale = reinterpret_cast<float4 *>(g_logscale_);
  using namespace gs;
  if (p.n < 0 || !loss || (p.n > 0 && (!p.logscale || !g_logscale)) || !(lambda_reg >= 0.f)) {
    set_error("gs_iso_reg: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  const int nblk = std::max(1, std::min(4 * 148, (p.n + kOptThreads - 1) / kOptThreads));
  if (!ws || ws_bytes < size_t(8) * nblk) {
    set_error("gs_iso_reg: workspace too small");
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  double *part = static_cast<double *>(ws);
  const float w = p.n > 0 ? lambda_reg / float(p.n) : 0.f;
  k_iso_reg<<<nblk, kOptThreads, 0, s>>>(reinterpret_cast<const float4 *>(p.logscale), p.n, w, g_logscale, part);
  k_iso_reg_final<<<1, kOptThreads, 0, s>>>(part, nblk, p.n, lambda_reg, loss);
  return check_launch("gs_iso_reg");
}

extern "C" int gs_adam_step(gs_params p, const float *g_mean_opa_, const float *g_quat_, const float *g_logscale_,
                            const float *g_rgb_, float *moments_, const gs_adam_cfg *cfg, gs_counters *cnt,
                            void *stream) {
  const float4 *g_mean_opa = reinterpret_cast<const float4 *>(g_mean_opa_);
  const float4 *g_quat = reinterpret_cast<const float4 *>(g_quat_);
  const float4 *g_logscale = reinterpret_cast<const float4 *>(g_logscale_);
  const float4 *g_rgb = reinterpret_cast<const float4 *>(g_rgb_);
  float4 *moments = reinterpret_cast<float4 *>(moments_);
  using namespace gs;
  if (p.n < 0 || !cfg || cfg->step < 1 || !(cfg->beta1 >= 0.0 && cfg->beta1 < 1.0) ||
      !(cfg->beta2 >= 0.0 && cfg->beta2 < 1.0) || !(cfg->eps > 0.0)) {
    set_error("gs_adam_step: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (p.n == 0) return GS_OK;
  if (!p.mean_opa || !p.quat || !p.logscale || !p.rgb || !g_mean_opa || !g_quat || !g_logscale || !g_rgb ||
      !moments) {
    set_error("gs_adam_step: null array");
    return GS_ERR_INVALID_ARG;
  }
  AdamArgs a;
  a.p[0] = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.mean_opa));
  a.p[1] = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.quat));
  a.p[2] = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.logscale));
  a.p[3] = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.rgb));
  a.g[0] = g_mean_opa;
  a.g[1] = g_quat;
  a.g[2] = g_logscale;
  a.g[3] = g_rgb;
  a.mv = moments;
  a.n = p.n;
  const float lm = cfg->lr_mean, lo = cfg->lr_opacity, lq = cfg->lr_quat, ls = cfg->lr_logscale, lc = cfg->lr_rgb;
  const float lr[4][4] = {{lm, lm, lm, lo}, {lq, lq, lq, lq}, {ls, ls, ls, 0.f}, {lc, lc, lc, 0.f}};
  for (int k = 0; k < 4; ++k)
    for (int c = 0; c < 4; ++c) a.lr[k][c] = lr[k][c];
  a.b1 = float(cfg->beta1);
  a.b2 = float(cfg->beta2);
  // 1 - beta from the fp64 betas (an fp32 0.999 would make it 0.00099998713)
  a.omb1 = float(1.0 - cfg->beta1);
  a.omb2 = float(1.0 - cfg->beta2);
  a.eps = float(cfg->eps);
  a.c1 = float(1.0 - std::pow(cfg->beta1, double(cfg->step)));
  a.c2 = float(1.0 - std::pow(cfg->beta2, double(cfg->step)));
  a.cnt = cnt;
  k_adam<<<(p.n + kOptThreads - 1) / kOptThreads, kOptThreads, 0, as_stream(stream)>>>(a);
  return check_launch("gs_adam_step");
}

extern "C" int gs_prune(gs_params p, const float *moments_, float o_thre, gs_params out, float *moments_out_,
                        void *ws, size_t ws_bytes, int32_t *n_out, void *stream) {
  const float4 *moments = reinterpret_cast<const float4 *>(moments_);
  float4 *moments_out = reinterpret_cast<float4 *>(moments_out_);
  using namespace gs;
  if (p.n < 0 || !n_out || !(o_thre > 0.f && o_thre < 1.f) || (moments != nullptr) != (moments_out != nullptr)) {
    set_error("gs_prune: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  const int nblk = std::max(1, (p.n + kOptThreads - 1) / kOptThreads);
  if (!ws || ws_bytes < size_t(4) * (nblk + 1)) {
    set_error("gs_prune: workspace too small");
    return GS_ERR_WORKSPACE;
  }
  if (p.n > 0 && (!p.mean_opa || !p.quat || !p.logscale || !p.rgb || !out.mean_opa || !out.quat ||
                  !out.logscale || !out.rgb)) {
    set_error("gs_prune: null array");
    return GS_ERR_INVALID_ARG;
  }
  cudaStream_t s = as_stream(stream);
  int *boff = static_cast<int *>(ws);
  const double lt = double(o_thre);
  if (p.n == 0) {
    cudaMemsetAsync(n_out, 0, sizeof(int32_t), s);
    return check_launch("gs_prune");
  }
  k_prune_count<<<nblk, kOptThreads, 0, s>>>(reinterpret_cast<const float4 *>(p.mean_opa), p.n, lt, boff);
  k_prune_scan<<<1, 1024, 0, s>>>(boff, nblk, n_out);
  PruneArgs a;
  const void *src[4] = {p.mean_opa, p.quat, p.logscale, p.rgb};
  const void *dst[4] = {out.mean_opa, out.quat, out.logscale, out.rgb};
  for (int k = 0; k < 4; ++k) {
    a.src[k] = reinterpret_cast<const float4 *>(src[k]);
    a.dst[k] = const_cast<float4 *>(reinterpret_cast<const float4 *>(dst[k]));
  }
  a.ms = moments;
  a.md = moments_out;
  a.n = p.n;
  a.lt = lt;
  a.boff = boff;
  k_prune_scatter<<<nblk, kOptThreads, 0, s>>>(a);
  return check_launch("gs_prune");
}
