// tracking_loss.cu — NEXT(1) gs_tracking_loss: the masked tracking loss of
// Eq. 15 (R29-R31).
//
//   L = sum_px M_inlier M_alpha (lambda_c e_c + (1 - lambda_c) e_d)
//   M_alpha  = alpha^3 (the "polynomial of the alpha map"; cube)
//   e_c      = (|dr| + |dg| + |db|) / 3, e_d = |D^ - D*|  (fp32, no contraction)
//   M_inlier = (D* > 0) & e_d <= mult * med(e_d) & e_c <= mult * med(e_c)
//              (medians over the valid pixels, lower median; mult = 50)
// The two medians are exact k-th order statistics found by an MSD radix
// select on the fp32 bit patterns (non-negative floats order as their bits):
// four 8-bit digit passes, each a kernel adding its blocks' histograms of
// the candidates sharing the prefix of the earlier digits into 16 replicas
// (few-way atomic contention); every block of the next kernel resolves the
// earlier digits itself from those complete histograms (no block waits on
// another, no extra launches).  Every decision is integer or fp32 with explicit
// rounding, so the masks are bit-deterministic; the loss value is an fp64
// fixed-order two-stage reduction.
#include <algorithm>

#include "gs_internal.cuh"

namespace gs {

constexpr int kTLThreads = 256;
constexpr int kTLPix = 4;       // pixels per thread (loads of all four issued first)
constexpr int kTLRep = 16;      // replicated global histograms per pass (block b adds into copy b % 16)

// workspace: [2][HW] keys, [4 passes][kTLRep][2][256] histograms (zeroed per
// call), per-block valid counts, fp64 partials, [8] state for k_tl_final
struct TLLayout {
  size_t keys, hist, nvalid, part, state, total;
};

static int tl_blocks(int64_t HW) { return int(std::max<int64_t>(1, (HW + kTLThreads * kTLPix - 1) / (kTLThreads * kTLPix))); }

static TLLayout tl_layout(int64_t HW) {
  TLLayout L;
  const int nblk = tl_blocks(HW);
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off = (off + b + 255) & ~size_t(255);
    return o;
  };
  L.keys = take(sizeof(uint32_t) * 2 * size_t(HW));
  L.hist = take(sizeof(uint32_t) * 4 * kTLRep * 512);
  L.nvalid = take(sizeof(uint32_t) * nblk);
  L.part = take(sizeof(double) * 2 * nblk);
  L.state = take(sizeof(uint32_t) * 8);
  L.total = off;
  return L;
}

struct TLArgs {
  const float *color, *depth, *alpha, *tc, *td;
  int64_t HW;
  float lambda_c, mult;
  uint32_t *keys;    // [0, HW) colour errors, [HW, 2HW) depth errors (0xffffffff = invalid pixel)
  uint32_t *hist;    // [pass][kTLRep][2][256]
  uint32_t *nvalid;  // [gridDim.x of the per-pixel kernels]
  double *part;
  uint32_t *state;   // (n, med_c bits, med_d bits) for k_tl_final
  float *loss, *g_color, *g_depth;
};

__device__ __forceinline__ float color_err(const TLArgs &a, int64_t q) {
  const float r0 = fabsf(__fsub_rn(__ldg(a.color + q), __ldg(a.tc + q)));
  const float r1 = fabsf(__fsub_rn(__ldg(a.color + a.HW + q), __ldg(a.tc + a.HW + q)));
  const float r2 = fabsf(__fsub_rn(__ldg(a.color + 2 * a.HW + q), __ldg(a.tc + 2 * a.HW + q)));
  return __fdiv_rn(__fadd_rn(__fadd_rn(r0, r1), r2), 3.f);
}

// Warp-aggregated shared-memory histogram increment: one atomic per distinct
// bin among the active lanes (the top digit of an error map is dominated by
// a few exponents, so plain atomics would serialise on them).
__device__ __forceinline__ void hist_add_agg(uint32_t *h, uint32_t bin, bool on) {
  unsigned todo = __ballot_sync(0xffffffffu, on);
  const int lane = threadIdx.x & 31;
  while (todo) {
    const int leader = __ffs(todo) - 1;
    const uint32_t b = __shfl_sync(0xffffffffu, bin, leader);
    const unsigned same = __ballot_sync(0xffffffffu, on && bin == b) & todo;
    if (lane == leader) atomicAdd(h + b, uint32_t(__popc(same)));
    todo &= ~same;
  }
}

// This block's shared histogram -> its replica of pass `pass` (few-way contention).
__device__ __forceinline__ void flush_hist(const TLArgs &a, const uint32_t *sh, int pass) {
  __syncthreads();
  uint32_t *g = a.hist + (size_t(pass) * kTLRep + blockIdx.x % kTLRep) * 512;
  for (int i = threadIdx.x; i < 512; i += blockDim.x)
    if (sh[i]) atomicAdd(g + i, sh[i]);
}

__device__ __forceinline__ uint32_t block_excl_scan_tl(uint32_t v, uint32_t *sh /* >= 33 */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = lane < int(blockDim.x >> 5) ? sh[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < int(blockDim.x >> 5)) sh[lane] = xi - x;
  }
  __syncthreads();
  const uint32_t r = inc - v + sh[w];
  __syncthreads();
  return r;
}

// The radix-select state after the digits of passes 0..last: every block
// recomputes it from the (complete) histograms of the earlier kernels, so no
// block waits on another.  k starts at floor((n - 1) / 2), the lower median's
// rank over the n valid pixels (R30).
struct SelState {
  uint32_t n, prefix[2], k[2];
};

__device__ SelState select_state(const TLArgs &a, int last) {
  static_assert(kTLThreads == 256, "one bin per thread and select");
  __shared__ uint32_t s_sh[2][33];
  __shared__ uint32_t s_pick[2][2];
  __shared__ uint32_t s_n;
  // the histogram counts of every pass this block needs, loaded up front
  uint32_t cnt[4][2];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int sel = 0; sel < 2; ++sel) {
      cnt[p][sel] = 0u;
      if (p <= last) {
        const uint32_t *g = a.hist + size_t(p) * kTLRep * 512 + 256 * sel + threadIdx.x;
#pragma unroll
        for (int r = 0; r < kTLRep; ++r) cnt[p][sel] += g[r * 512];
      }
    }
  uint32_t n = 0;
  for (int b = threadIdx.x; b < int(gridDim.x); b += blockDim.x) n += a.nvalid[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_n, n);
  __syncthreads();
  SelState st;
  st.n = s_n;
  st.prefix[0] = st.prefix[1] = 0u;
  st.k[0] = st.k[1] = st.n ? (st.n - 1) / 2 : 0u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    if (p > last) break;
    // exclusive scans of both selects' counts over the 256 digits
    uint32_t inc[2] = {cnt[p][0], cnt[p][1]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int sel = 0; sel < 2; ++sel) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc[sel], o);
        if (lane >= o) inc[sel] += y;
      }
    }
    if (lane == 31) {
      s_sh[0][w] = inc[0];
      s_sh[1][w] = inc[1];
    }
    __syncthreads();
    if (w < 2) {  // warp `w` scans select w's 8 warp totals
      const uint32_t x = lane < 8 ? s_sh[w][lane] : 0u;
      uint32_t xi = x;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      if (lane < 8) s_sh[w][lane] = xi - x;
    }
    __syncthreads();
#pragma unroll
    for (int sel = 0; sel < 2; ++sel) {
      const uint32_t c = cnt[p][sel], ex = inc[sel] - c + s_sh[sel][w];
      // the digit whose [ex, ex + c) holds rank k (digit 255 if the counts run short)
      if ((ex <= st.k[sel] && st.k[sel] < ex + c) || (threadIdx.x == 255 && ex + c <= st.k[sel])) {
        s_pick[sel][0] = threadIdx.x;
        s_pick[sel][1] = ex;
      }
    }
    __syncthreads();
#pragma unroll
    for (int sel = 0; sel < 2; ++sel) {
      st.prefix[sel] |= s_pick[sel][0] << (24 - 8 * p);
      st.k[sel] -= s_pick[sel][1];
    }
    __syncthreads();
  }
  return st;
}

// Pass 0: errors -> keys, valid counts, histograms of the top digit.
__global__ void __launch_bounds__(kTLThreads) k_tl_resid(TLArgs a) {
  __shared__ uint32_t sh[2][256];
  __shared__ uint32_t s_nv;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&sh[0][0])[i] = 0u;
  if (threadIdx.x == 0) s_nv = 0;
  __syncthreads();
  uint32_t kc[kTLPix], kd[kTLPix];
  bool ok[kTLPix];
  uint32_t nv = 0;
  const int64_t q0 = int64_t(blockIdx.x) * (kTLThreads * kTLPix) + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kTLPix; ++i) {
    const int64_t q = q0 + i * kTLThreads;
    const float t = q < a.HW ? __ldg(a.td + q) : 0.f;
    ok[i] = t > 0.f;
    kc[i] = kd[i] = 0xffffffffu;
    if (ok[i]) {
      kc[i] = __float_as_uint(color_err(a, q));
      kd[i] = __float_as_uint(fabsf(__fsub_rn(__ldg(a.depth + q), t)));
      ++nv;
    }
  }
#pragma unroll
  for (int i = 0; i < kTLPix; ++i) {
    const int64_t q = q0 + i * kTLThreads;
    hist_add_agg(sh[0], kc[i] >> 24, ok[i]);
    hist_add_agg(sh[1], kd[i] >> 24, ok[i]);
    if (q < a.HW) {
      a.keys[q] = kc[i];
      a.keys[a.HW + q] = kd[i];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nv += __shfl_xor_sync(0xffffffffu, nv, o);
  if ((threadIdx.x & 31) == 0 && nv) atomicAdd(&s_nv, nv);
  flush_hist(a, &sh[0][0], 0);
  if (threadIdx.x == 0) a.nvalid[blockIdx.x] = s_nv;
}

// Passes 1..3: histograms of digit `pass` over the keys matching the prefix
// of the earlier digits.
__global__ void __launch_bounds__(kTLThreads) k_tl_hist(TLArgs a, int pass) {
  __shared__ uint32_t sh[2][256];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) (&sh[0][0])[i] = 0u;
  const int64_t q0 = int64_t(blockIdx.x) * (kTLThreads * kTLPix) + threadIdx.x;
  uint32_t kc[kTLPix], kd[kTLPix];
#pragma unroll
  for (int i = 0; i < kTLPix; ++i) {  // loads in flight while the digits are resolved
    const int64_t q = q0 + i * kTLThreads;
    kc[i] = q < a.HW ? a.keys[q] : 0xffffffffu;
    kd[i] = q < a.HW ? a.keys[a.HW + q] : 0xffffffffu;
  }
  const SelState st = select_state(a, pass - 1);
  const int shift = 24 - 8 * pass;
  const uint32_t hi_mask = 0xffffffffu << (shift + 8);
#pragma unroll
  for (int i = 0; i < kTLPix; ++i) {
    if (kc[i] != 0xffffffffu && (kc[i] & hi_mask) == st.prefix[0]) atomicAdd(&sh[0][(kc[i] >> shift) & 255u], 1u);
    if (kd[i] != 0xffffffffu && (kd[i] & hi_mask) == st.prefix[1]) atomicAdd(&sh[1][(kd[i] >> shift) & 255u], 1u);
  }
  flush_hist(a, &sh[0][0], pass);
}

__device__ __forceinline__ double block_sum_tl(double v, double *sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// Masks, gradient maps and per-block fp64 partials of the loss.
__global__ void __launch_bounds__(kTLThreads) k_tl_apply(TLArgs a) {
  __shared__ double sh[kTLThreads];
  const SelState st = select_state(a, 3);
  const bool any = st.n > 0;
  const float med_c = __uint_as_float(st.prefix[0]), med_d = __uint_as_float(st.prefix[1]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.state[0] = st.n;
    a.state[1] = st.prefix[0];
    a.state[2] = st.prefix[1];
  }
  const float thr_c = __fmul_rn(a.mult, med_c), thr_d = __fmul_rn(a.mult, med_d);
  const float gc_scale = __fdiv_rn(a.lambda_c, 3.f), gd_scale = __fsub_rn(1.f, a.lambda_c);
  double acc = 0.0, ninl = 0.0;
  const int64_t q0 = int64_t(blockIdx.x) * (kTLThreads * kTLPix) + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kTLPix; ++i) {
    const int64_t q = q0 + i * kTLThreads;
    if (q >= a.HW) break;
    const uint32_t kc = a.keys[q], kd = a.keys[a.HW + q];
    const bool inl = any && kc != 0xffffffffu && __uint_as_float(kd) <= thr_d && __uint_as_float(kc) <= thr_c;
    const float al = __ldg(a.alpha + q);
    const float w = inl ? __fmul_rn(__fmul_rn(al, al), al) : 0.f;  // M_inlier M_alpha
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float r = __fsub_rn(__ldg(a.color + ch * a.HW + q), __ldg(a.tc + ch * a.HW + q));
      a.g_color[ch * a.HW + q] = __fmul_rn(__fmul_rn(w, gc_scale), float((r > 0.f) - (r < 0.f)));
    }
    float gd = 0.f;
    if (inl) {
      const float r = __fsub_rn(__ldg(a.depth + q), __ldg(a.td + q));
      gd = __fmul_rn(__fmul_rn(w, gd_scale), float((r > 0.f) - (r < 0.f)));
      acc += double(w) * (double(a.lambda_c) * double(__uint_as_float(kc)) +
                          (1.0 - double(a.lambda_c)) * double(__uint_as_float(kd)));
      ninl += 1.0;
    }
    a.g_depth[q] = gd;
  }
  acc = block_sum_tl(acc, sh);
  ninl = block_sum_tl(ninl, sh);
  if (threadIdx.x == 0) {
    a.part[2 * blockIdx.x] = acc;
    a.part[2 * blockIdx.x + 1] = ninl;
  }
}

__global__ void __launch_bounds__(kTLThreads) k_tl_final(TLArgs a, int nblk) {
  __shared__ double sh[kTLThreads];
  double acc = 0.0, ninl = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {  // fixed order per thread
    acc += a.part[2 * b];
    ninl += a.part[2 * b + 1];
  }
  acc = block_sum_tl(acc, sh);
  ninl = block_sum_tl(ninl, sh);
  if (threadIdx.x == 0) {
    const bool any = a.state[0] > 0;
    a.loss[0] = float(acc);
    a.loss[1] = any ? __uint_as_float(a.state[1]) : 0.f;
    a.loss[2] = any ? __uint_as_float(a.state[2]) : 0.f;
    a.loss[3] = float(ninl);
  }
}

}  // namespace gs

extern "C" size_t gs_tracking_loss_workspace_bytes(gs_camera cam) {
  if (!gs::camera_ok(cam)) return 0;
  return gs::tl_layout(int64_t(cam.width) * cam.height).total;
}

extern "C" int gs_tracking_loss(gs_camera cam, const float *color, const float *depth, const float *alpha,
                                const float *tgt_color, const float *tgt_depth, float lambda_c, float inlier_mult,
                                void *ws, size_t ws_bytes, float *loss, float *dL_dcolor, float *dL_ddepth,
                                void *stream) {
  using namespace gs;
  if (!camera_ok(cam) || !color || !depth || !alpha || !tgt_color || !tgt_depth || !loss || !dL_dcolor ||
      !dL_ddepth || !(lambda_c >= 0.f && lambda_c <= 1.f) || !(inlier_mult > 0.f)) {
    set_error("gs_tracking_loss: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  const int64_t HW = int64_t(cam.width) * cam.height;
  const TLLayout L = tl_layout(HW);
  if (!ws || ws_bytes < L.total) {
    set_error("gs_tracking_loss: workspace %zu < %zu bytes", ws_bytes, L.total);
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char *w = static_cast<char *>(ws);
  TLArgs a{color, depth, alpha, tgt_color, tgt_depth, HW, lambda_c, inlier_mult,
           reinterpret_cast<uint32_t *>(w + L.keys), reinterpret_cast<uint32_t *>(w + L.hist),
           reinterpret_cast<uint32_t *>(w + L.nvalid), reinterpret_cast<double *>(w + L.part),
           reinterpret_cast<uint32_t *>(w + L.state), loss, dL_dcolor, dL_ddepth};
  cudaMemsetAsync(w + L.hist, 0, sizeof(uint32_t) * 4 * kTLRep * 512, s);
  const int nblk = tl_blocks(HW);
  k_tl_resid<<<nblk, kTLThreads, 0, s>>>(a);
  for (int pass = 1; pass < 4; ++pass) k_tl_hist<<<nblk, kTLThreads, 0, s>>>(a, pass);
  k_tl_apply<<<nblk, kTLThreads, 0, s>>>(a);
  k_tl_final<<<1, kTLThreads, 0, s>>>(a, nblk);
  return check_launch("gs_tracking_loss");
}
