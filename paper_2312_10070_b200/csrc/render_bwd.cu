// render_bwd.cu — S5 + S6 gs_render_bwd (Eqs. 7-8).
//
// S5 (k_bwd_pixels): one CTA (2 warps) per tile, 4 pixels of a row per
// thread, each warp a 16x8 strip.  Every pixel replays its composited entries
// back to front starting from T_final and n_contrib, recomputing alpha with
// the very same entry/row terms and pair exponent as gs_render_fwd (H5),
// reconstructing T_j = T_{j+1}/(1-alpha_j) and carrying the suffix form of
// Eq. 8 (one scalar Q = G . S per pixel).  The per-pixel arithmetic runs on
// fp32x2 pixel pairs (FFMA2).  Each warp walks, back to front, the compacted
// list of staged entries that meet its strip, two entries per step (their
// decisions, alphas and reciprocals first, then the T / Q chain of each);
// per (thread, entry) the 2-D gradients are summed over the thread's pixels,
// then across the warp through a per-warp shared-memory slab (skipped when no
// lane composited the entry, replaced by direct vector reds when <= 2 lanes
// did) and added to the grad2d scratch.
//
// S6 (k_bwd_gauss): one thread per visible Gaussian chains the 2-D gradients
// to mean, quaternion, log-scales, opacity logit and colour ("derived as in
// [kerbl]"), and for tracking reduces the pose partials block-wise.
#include "raster_common.cuh"

namespace gs {

// grad2d record [n][12]: (u, v, A, B), (C, p_z, logit, 0), (r, g, b, 0)
constexpr int kG2 = 12;
#ifndef GAUSS_THREADS
#define GAUSS_THREADS 128
#endif
constexpr int kGaussThreads = GAUSS_THREADS;  // k_bwd_gauss block (one pose-partial record per block)

struct BwdArgs {
  const double2 *uv;
  const float4 *coef;
  const float4 *rgbz;
  const float4 *conic_o;
  const int32_t *sorted_idx;
  const int2 *tile_range;
  const int32_t *tile_order;
  const float *T_final;
  const int32_t *n_contrib;
  const float *dL_dcolor, *dL_ddepth, *dL_dalpha;
  int W, H, TX;
  float *grad2d;
  uint32_t *tile_done;  // nullable: [T + 1], wait for (and re-arm) the forward's per-tile flag
  int T;                // tiles; tile_done[T] counts timed-out waits
  int n;                // Gaussians (bounds checks of the debug build)
};

__device__ __forceinline__ void red_add_v4(float *addr, float x, float y, float z, float w) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(x), "f"(y), "f"(z), "f"(w)
               : "memory");
}

constexpr int kBPX = 4;   // pixels per thread in the backward (two fp32x2 pairs)
#ifndef BWD_MINB
#define BWD_MINB 1
#endif
constexpr int kBwdMinBlocks = BWD_MINB;  // resident CTAs per SM the register budget must allow
// at most this many contributing lanes: per-lane vector reds instead of the
// shared-memory slab.  Re-tuned at the end of round 2 (the faster binning
// changed what overlaps the backward): mapping 20 — k_bwd_pixels alone 170 /
// 168 / 164 / 164 µs and the step 2382 / 2398 / 2421 / 2420 MP/s for 4 / 8 /
// 20 / 24, all 32 lanes direct 340 µs (every lane's reds on one record
// contend in L2); pose-only 24 — 2765 / 2776 / 2788 / 2467 it/s for 16 / 20 /
// 24 / 32)
#ifndef BWD_OMA2
#define BWD_OMA2 1
#endif
#ifndef BWD_DIRECT
#define BWD_DIRECT 20
#endif
#ifndef BWD_DIRECT_POSE
#define BWD_DIRECT_POSE 24
#endif
using BG = Geo<kBPX, 16>;  // 2 warps, 16x8 pixel strips

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 bcast(float x) { return make_float2(x, x); }

// per-thread backward state of its 4 pixels (two fp32x2 pairs): T
// (reconstructed back to front), upstream G, and the single suffix scalar
// Q = G . S of Eq. 8's accumulators S = (S_C, S_D, S_A):
//   dL/dalpha_j = T_j (G . X_j - Q),  Q <- Q + alpha_j (G . X_j - Q)
struct BwdPix {
  float2 T[2], G0[2], G1[2], G2[2], GD[2], GA[2], Q[2];
  int last[kBPX];
};

// Geometry of the per-warp reduction slab of bwd_entry: NV values per entry
// (10 for mapping; 6 = u, v, A, B, C, p_z for the pose-only backward), L
// lanes per value, each summing R rows (row stride NV + 1, odd: conflict-free
// stores); rows 32 .. L R - 1 are zero padding.
template <bool kParams>
struct Slab {
  static constexpr int NV = kParams ? 10 : 6;
  static constexpr int L = 32 / NV;
  static constexpr int R = (32 + L - 1) / L;
  static constexpr int S = NV + 1;
  static constexpr int SIZE = L * R * S;
};

// per-lane roles in the shared-memory reduction of bwd_entry: lane L v + p
// (v < NV, p < L) sums value v over the slab rows = p mod L; lane L v writes
// the total, scaled by wsc, to grad2d[woff]
struct RedRole {
  const float *col;  // first slab row of this lane's column
  int woff;          // grad2d record offset of value v
  float wsc;         // sign of the value and the 1/2 of dsigma/dA, dsigma/dC
  bool writer;
};

// One list entry j at the thread's pixels: alpha replay (H5), T by division
// (R16), Eq. 8 through Q, per-thread sums, then the warp reduction into
// grad2d.  Branch-free per pixel: alpha = 0 leaves T and Q unchanged and
// contributes exact zeros.  pass[k]: the pixel's decision (entry inside its
// n_contrib and alpha~ >= 1/255, the forward's e >= kExpMin, R2'); any: one
// of this lane's pixels passes; ball: the warp's ballot of `any` (nonzero).
// acc layout (before the writer's sign/scale): 0 u, 1 v, 2 A-term, 3 B,
// 4 C-term, 5 p_z, 6 logit, 7 r, 8 g, 9 b
// alpha of an entry at the thread's pixel pairs (the forward's value, H5; a
// skipped pixel's exponent becomes -inf: alpha = 0), 1 / (1 - alpha) (R16) and
// the alpha that carries a gradient (0 where clamped, R17): independent of
// the T / Q chain, so computed for both entries of a step up front
struct AlphaPrep {
  float2 al[2], ir[2], ag[2];
};

__device__ __forceinline__ AlphaPrep alpha_prep(const float2 e[2], const bool pass[kBPX]) {
  AlphaPrep p;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float a0 = fminf(ex2_approx(pass[2 * h] ? e[h].x : -INFINITY), kAlphaMax);
    const float a1 = fminf(ex2_approx(pass[2 * h + 1] ? e[h].y : -INFINITY), kAlphaMax);
    p.al[h] = make_float2(a0, a1);
#if BWD_OMA2
    const float2 oma = __fadd2_rn(make_float2(1.f, 1.f), make_float2(-a0, -a1));  // 1 - alpha as one FADD2
    p.ir[h] = make_float2(rcp_approx(oma.x), rcp_approx(oma.y));
#else
    p.ir[h] = make_float2(rcp_approx(1.f - a0), rcp_approx(1.f - a1));
#endif
    p.ag[h] = make_float2(e[h].x < kExpClamp ? a0 : 0.f, e[h].y < kExpClamp ? a1 : 0.f);
  }
  return p;
}

template <bool kParams>
__device__ __forceinline__ void bwd_entry(BwdPix &s, const AlphaPrep &ap, bool any,
                                          unsigned ball, float4 c, float4 cn, float2 ul, float fpy,
                                          const float2 fx[2], float *dst, float *red, const RedRole &rr) {
  const float dy = ul.y - fpy;  // Delta = mu^I - pixel; one row: dy is shared
  // per-thread sums over its pixels (as pair sums) of ga = alpha dL/dalpha
  // (0 if clamped) and ga dx, ga dx^2; dsigma/d(u, v, A, B, C) and
  // dalpha/dlogit are formed once per (thread, entry) from them, the conic,
  // dy and o (entry constants)
  float2 ga[2], t[2], wt[2], dx[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float2 al = ap.al[h];
    // T_j = T_{j+1} / (1 - alpha_j) (R16)
    s.T[h] = __fmul2_rn(s.T[h], ap.ir[h]);
    wt[h] = __fmul2_rn(al, s.T[h]);
    // Eq. 8 chained with Eq. 7 through the suffix scalar Q
    const float2 gx = __ffma2_rn(
        s.G0[h], bcast(c.x), __ffma2_rn(s.G1[h], bcast(c.y), __ffma2_rn(s.G2[h], bcast(c.z), __ffma2_rn(s.GD[h], bcast(c.w), s.GA[h]))));
    const float2 d = __fadd2_rn(gx, make_float2(-s.Q[h].x, -s.Q[h].y));
    const float2 galpha = __fmul2_rn(s.T[h], d);
    s.Q[h] = __ffma2_rn(al, d, s.Q[h]);
    // clamped alpha (alpha~ >= 0.999: e >= kExpClamp): no gradient (R17)
    ga[h] = __fmul2_rn(ap.ag[h], galpha);
    dx[h] = __fadd2_rn(bcast(ul.x), make_float2(-fx[h].x, -fx[h].y));
    t[h] = __fmul2_rn(ga[h], dx[h]);
  }
  const float2 sga = __fadd2_rn(ga[0], ga[1]);
  const float2 sgx = __fadd2_rn(t[0], t[1]);
  const float2 sgxx = __ffma2_rn(t[1], dx[1], __fmul2_rn(t[0], dx[0]));
  const float2 sz = __ffma2_rn(wt[1], s.GD[1], __fmul2_rn(wt[0], s.GD[0]));  // dD/dz_j = alpha_j T_j
  const float Sga = sga.x + sga.y, Sgx = sgx.x + sgx.y;
  // dalpha/dsigma = -alpha, dsigma/du = A dx + B dy, dsigma/dv = B dx + C dy,
  // dsigma/d(A, B, C) = (dx^2/2, dx dy, dy^2/2), dalpha/dlogit = alpha (1 - o);
  // the signs of values 0-4 and the halves are applied by the writer (wsc)
  float acc[10];
  acc[0] = fmaf(cn.x, Sgx, cn.y * dy * Sga);
  acc[1] = fmaf(cn.y, Sgx, cn.z * dy * Sga);
  acc[2] = sgxx.x + sgxx.y;
  acc[3] = dy * Sgx;
  acc[4] = dy * dy * Sga;
  acc[5] = sz.x + sz.y;
  acc[6] = kParams ? (1.f - cn.w) * Sga : 0.f;
  if (kParams) {  // dC/dc_j = alpha_j T_j
    const float2 sr = __ffma2_rn(wt[1], s.G0[1], __fmul2_rn(wt[0], s.G0[0]));
    const float2 sg = __ffma2_rn(wt[1], s.G1[1], __fmul2_rn(wt[0], s.G1[0]));
    const float2 sb = __ffma2_rn(wt[1], s.G2[1], __fmul2_rn(wt[0], s.G2[0]));
    acc[7] = sr.x + sr.y;
    acc[8] = sg.x + sg.y;
    acc[9] = sb.x + sb.y;
  } else {
    acc[7] = acc[8] = acc[9] = 0.f;
  }
  if (__popc(ball) <= (kParams ? BWD_DIRECT : BWD_DIRECT_POSE)) {  // few lanes: write directly
    if (any) {
      // grad2d record: (u, v, A, B), (C, p_z, logit, 0), (r, g, b, 0)
      red_add_v4(dst, -acc[0], -acc[1], -0.5f * acc[2], -acc[3]);
      red_add_v4(dst + 4, -0.5f * acc[4], acc[5], acc[6], 0.f);
      if (kParams) red_add_v4(dst + 8, acc[7], acc[8], acc[9], 0.f);
    }
    return;
  }
  // through this warp's shared-memory slab (Slab): lane l stores its NV
  // values in row l; lane L v + p sums value v over the rows = p mod L
  // (zero rows past 32: no bounds checks), the L partial sums meet by
  // shuffles, lane L v adds the total to grad2d
  using SL = Slab<kParams>;
  const int lane = threadIdx.x & 31;
  float *row = red + lane * SL::S;
  __syncwarp();  // the previous entry's reads of the slab are done
#pragma unroll
  for (int v = 0; v < SL::NV; ++v) row[v] = acc[v];
  __syncwarp();
  float cs[SL::R];
#pragma unroll
  for (int t = 0; t < SL::R; ++t) cs[t] = rr.col[t * SL::L * SL::S];
  float part;
  if (SL::R == 11) {  // pairwise (depth 4, not a chain of dependent adds)
    part = (((cs[0] + cs[1]) + (cs[2] + cs[3])) + ((cs[4] + cs[5]) + (cs[6] + cs[7]))) + ((cs[8] + cs[9]) + cs[10]);
  } else {
    part = cs[0];
#pragma unroll
    for (int t = 1; t < SL::R; t += 2) part += t + 1 < SL::R ? cs[t] + cs[t + 1] : cs[t];
  }
  if (SL::L == 3) {
    part += __shfl_down_sync(0xffffffffu, part, 1) + __shfl_down_sync(0xffffffffu, part, 2);
  } else {  // L = 5: (x0 + x1) + (x2 + x3) + x4 on the group's first lane
    float q = part + __shfl_down_sync(0xffffffffu, part, 1);
    q += __shfl_down_sync(0xffffffffu, q, 2);
    part = q + __shfl_down_sync(0xffffffffu, part, 4);
  }
  if (rr.writer) atomicAdd(dst + rr.woff, rr.wsc * part);
}

// one staged list entry of the backward
struct __align__(16) BwdRec {
  float4 p;      // entry terms (a', b', d', K)
  float4 rgbz;   // colour, camera depth
  float4 conic;  // (A, B, C, o)
  float2 q;      // (DV, log2 o)
  float2 uv;     // tile-local mean
  int idx, pad[3];
};

template <bool kParams, bool kAlphaUp>
__global__ void __launch_bounds__(BG::kThreads, kBwdMinBlocks) k_bwd_pixels(BwdArgs a) {
  // one staged record per entry (one base address + immediate offsets);
  // record kBatch is a sentinel entry whose exponent is -inf
  __shared__ BwdRec s_rec[kBatch + 1];
  __shared__ unsigned char s_mask[kBatch];
  __shared__ unsigned char s_list[BG::kWarps][kBatch + 2];
  __shared__ int s_lmax;
  __shared__ float s_red[BG::kWarps][Slab<kParams>::SIZE];  // per-warp reduction slabs (rows >= 32 are 0)
  // with tile_done the forward's per-tile flags order this kernel after its
  // tile; else wait for the preceding grid (PDL; a no-op without it)
  if (!a.tile_done) pdl_wait();
  pdl_trigger();
  const int tile = a.tile_order ? __ldg(a.tile_order + blockIdx.x) : int(blockIdx.x);
  GS_ASSERT(tile >= 0 && tile < a.T);
  if (a.tile_done) {
    // launched programmatically dependent on gs_render_fwd_l1: every forward
    // CTA has started (launch_dependents), so this tile's flag is set in
    // bounded time; the wait is capped (~0.4 s) so a misuse cannot hang, and
    // a timeout is counted in tile_done[T] (the flag is then left as it is)
    if (threadIdx.x == 0) {
      uint32_t f = 0;
      for (long long it = 0; it < (1ll << 22); ++it) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(a.tile_done + tile) : "memory");
        if (f) break;
        __nanosleep(100);
      }
      if (f)
        a.tile_done[tile] = 0u;  // re-armed for the next forward
      else
        atomicAdd(a.tile_done + a.T, 1u);
    }
    __syncthreads();
  }
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int w = threadIdx.x >> 5;
  const PixGeom pg = pix_geom<BG>(tx, ty, a.H);
  const double ox = double(tx * kTile), oy = double(ty * kTile);
  const int2 range = a.tile_range[tile];
  GS_ASSERT(range.x >= 0 && range.x <= range.y);
  const size_t HW = size_t(a.W) * a.H;
  const float2 fx[2] = {make_float2(pg.fpx0, pg.fpx0 + 1.f), make_float2(pg.fpx0 + 2.f, pg.fpx0 + 3.f)};
  BwdPix s;
  int tmax = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float t[2] = {1.f, 1.f}, g0[2] = {0.f, 0.f}, g1[2] = {0.f, 0.f}, g2[2] = {0.f, 0.f}, gd[2] = {0.f, 0.f},
          ga[2] = {0.f, 0.f};
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int k = 2 * h + m;
      s.last[k] = 0;
      if (pg.row_in && pg.px0 + k < a.W) {
        const size_t q = size_t(pg.py) * a.W + pg.px0 + k;
        t[m] = a.T_final[q];
        s.last[k] = a.n_contrib[q];
        GS_ASSERT(s.last[k] >= 0 && s.last[k] <= range.y - range.x);
        g0[m] = a.dL_dcolor[q];
        g1[m] = a.dL_dcolor[HW + q];
        g2[m] = a.dL_dcolor[2 * HW + q];
        gd[m] = a.dL_ddepth[q];
        if (kAlphaUp) ga[m] = a.dL_dalpha[q];
        tmax = max(tmax, s.last[k]);
      }
    }
    s.T[h] = make_float2(t[0], t[1]);
    s.G0[h] = make_float2(g0[0], g0[1]);
    s.G1[h] = make_float2(g1[0], g1[1]);
    s.G2[h] = make_float2(g2[0], g2[1]);
    s.GD[h] = make_float2(gd[0], gd[1]);
    s.GA[h] = make_float2(ga[0], ga[1]);
    s.Q[h] = make_float2(0.f, 0.f);
  }
  if (threadIdx.x == 0) {
    s_lmax = 0;
    s_rec[kBatch].p = make_float4(0.f, 0.f, 0.f, 0.f);
    s_rec[kBatch].q = make_float2(0.f, -INFINITY);
  }
  {
    using SL = Slab<kParams>;
    constexpr int kPad = SL::SIZE - 32 * SL::S;
    for (int i = threadIdx.x; i < BG::kWarps * kPad; i += blockDim.x) s_red[i / kPad][32 * SL::S + i % kPad] = 0.f;
  }
  __syncthreads();
  // warp-level bound: entries at or beyond every lane's n_contrib are skipped
  int wmax = tmax;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  if ((threadIdx.x & 31) == 0 && wmax > 0) atomicMax(&s_lmax, wmax);
  __syncthreads();
  const int lmax = s_lmax;
  unsigned char *list = s_list[w];
  RedRole rr;
  {
    using SL = Slab<kParams>;
    const int lane = threadIdx.x & 31, rv = lane / SL::L, rp = lane % SL::L;
    rr.col = s_red[w] + rp * SL::S + rv;  // lanes past NV L read the padding column and never write
    rr.woff = rv < 7 ? rv : rv + 1;
    rr.wsc = (rv == 2 || rv == 4) ? -0.5f : (rv < 4 ? -1.f : 1.f);
    rr.writer = lane < SL::NV * SL::L && rp == 0;
  }
  for (int end = lmax; end > 0; end -= kBatch) {
    const int beg = max(end - kBatch, 0);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < BG::kRecPerThread; ++r) {
      const int i = r * BG::kThreads + threadIdx.x;
      const int k = beg + i;
      if (k < end) {
        const int g = __ldg(a.sorted_idx + range.x + k);
        GS_ASSERT(g >= 0 && g < a.n);
        const double2 u = __ldg(a.uv + g);
        const float4 cf = __ldg(a.coef + g);
        const float ul = float(u.x - ox), vl = float(u.y - oy);
        const EntryTerms et = entry_terms(cf, ul, vl);
        BwdRec &rc = s_rec[i];
        rc.p = et.p;
        rc.q = et.q;
        rc.uv = make_float2(ul, vl);
        rc.rgbz = __ldg(a.rgbz + g);
        rc.conic = __ldg(a.conic_o + g);
        rc.idx = g;
        s_mask[i] = (unsigned char)entry_block_mask<BG>(cf, ul, vl);
      }
    }
    __syncthreads();
    // back to front over this warp's hits, two per step (their exponents are
    // independent; the entries are replayed in order).  Entries missing the
    // warp's strip cannot pass the exponent pre-test at any of its pixels.
    // Hits are list[1..nh]; list[0] is the sentinel.
    if ((threadIdx.x & 31) == 0) list[0] = (unsigned char)kBatch;
    const int nh = warp_hit_list(s_mask, min(end, wmax) - beg, list + 1, kBatch);
    // the next pair's list indices and entry terms are loaded one step ahead
    // (list[0] is the sentinel: indices below 0 are clamped to it)
    int ja = list[nh], jb = list[max(nh - 1, 0)];
    float4 pa = s_rec[ja].p, pb = s_rec[jb].p;
    float2 qa = s_rec[ja].q, qb = s_rec[jb].q;
    for (int kk = nh; kk >= 1; kk -= 2) {
      const RowTerms ra = row_terms(pa, qa, pg.fpy);
      const RowTerms rb = row_terms(pb, qb, pg.fpy);
      const int ja_ = ja, jb_ = jb;
      ja = list[max(kk - 2, 0)];
      jb = list[max(kk - 3, 0)];
      pa = s_rec[ja].p;
      pb = s_rec[jb].p;
      qa = s_rec[ja].q;
      qb = s_rec[jb].q;
      float2 ea[2], eb[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ea[h] = pair_exponent(ra, fx[h]);
        eb[h] = pair_exponent(rb, fx[h]);
      }
      // decisions and alphas of both entries first (independent of the T / Q chain)
      bool pass[2][kBPX], any[2];
      unsigned ball[2];
      AlphaPrep ap[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int pos = beg + (u ? jb_ : ja_);  // entry position in the tile list
        const float2 *e = u ? eb : ea;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          pass[u][2 * h] = pos < s.last[2 * h] && e[h].x >= kExpMin;
          pass[u][2 * h + 1] = pos < s.last[2 * h + 1] && e[h].y >= kExpMin;
        }
        any[u] = pass[u][0] || pass[u][1] || pass[u][2] || pass[u][3];
        ball[u] = __ballot_sync(0xffffffffu, any[u]);
        ap[u] = alpha_prep(e, pass[u]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!ball[u]) continue;
        const BwdRec &rc = s_rec[u ? jb_ : ja_];
        bwd_entry<kParams>(s, ap[u], any[u], ball[u], rc.rgbz, rc.conic, rc.uv, pg.fpy, fx,
                           a.grad2d + size_t(rc.idx) * kG2, s_red[w], rr);
      }
    }
  }
}

struct GaussArgs {
  gs_params p;
  const gs_view *view;
  float fx, fy;
  const float4 *conic_o;
  const int32_t *tiles_touched;
  float *grad2d;
  float4 *g_mean_opa, *g_quat, *g_logscale, *g_rgb;
  float *pose_partials;
  bool atomic_acc;  // GS_BWD_ATOMIC_ACC: g_* += by red.global.add.v4
};

// S6 CTAs per SM (128 threads): 5 (with the fp64 chain's spills) measured
// best with FWD_MINB 8, 2446 -> 2458 MP/s; 6 slower
#ifndef GAUSS_MINB
#define GAUSS_MINB 5
#endif
template <bool kParams, bool kPose>
__global__ void __launch_bounds__(kGaussThreads, GAUSS_MINB) k_bwd_gauss(GaussArgs a) {
  // the view in fp64, once per block (exact)
  __shared__ double sV[12];
  if (threadIdx.x < 12) sV[threadIdx.x] = double(__ldg(threadIdx.x < 9 ? &a.view->R[threadIdx.x] : &a.view->t[threadIdx.x - 9]));
  __syncthreads();
  pdl_begin();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float pose[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) pose[k] = 0.f;
  // all loads are issued up front (one DRAM round trip per thread, not three)
  const bool inb = i < a.p.n;
  const int tt = inb ? __ldg(a.tiles_touched + i) : 0;
  float4 mo = make_float4(0.f, 0.f, 0.f, 0.f), qf = mo, lf = mo, cn = mo, ga = mo, gb = mo, gc = mo;
  float4 old_m = mo, old_q = mo, old_l = mo, old_c = mo;
  float4 *g2 = reinterpret_cast<float4 *>(a.grad2d) + 3 * size_t(inb ? i : 0);
  if (inb) {
    mo = __ldg(reinterpret_cast<const float4 *>(a.p.mean_opa) + i);
    qf = __ldg(reinterpret_cast<const float4 *>(a.p.quat) + i);
    lf = __ldg(reinterpret_cast<const float4 *>(a.p.logscale) + i);
    cn = __ldg(a.conic_o + i);
    ga = g2[0];
    gb = g2[1];
    if (kParams) {
      gc = g2[2];
      if (!a.atomic_acc) {
        old_m = a.g_mean_opa[i];
        old_q = a.g_quat[i];
        old_l = a.g_logscale[i];
        old_c = a.g_rgb[i];
      }
    }
  }
  if (tt > 0) {
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    g2[0] = z4;  // leave the scratch zeroed for the next call
    g2[1] = z4;
    if (kParams) g2[2] = z4;
    // The chain of P:172 in fp64: it is ~600 flops per Gaussian in a kernel
    // bound by HBM, and fp32 loses digits to cancellation (e.g. the
    // log-scale term of small splats, the tangent projection of dL/dq).
    double R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = sV[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = sV[9 + k];
    const double gu = ga.x, gv = ga.y, gA = ga.z, gB = ga.w, gC = gb.x, gz = gb.y;
    const double mu[3] = {mo.x, mo.y, mo.z};
    double p[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) p[r] = R[3 * r] * mu[0] + R[3 * r + 1] * mu[1] + R[3 * r + 2] * mu[2] + t[r];
    const double x = p[0], y = p[1], z = p[2];
    // Sigma = M M^T, M = R_q S
    const double q0 = qf.x, q1 = qf.y, q2 = qf.z, q3 = qf.w;
    const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const double iq = 1.0 / qn;
    const double qw = q0 * iq, qx = q1 * iq, qy = q2 * iq, qz = q3 * iq;
    double Rq[9];
    Rq[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
    Rq[1] = 2.0 * (qx * qy - qw * qz);
    Rq[2] = 2.0 * (qx * qz + qw * qy);
    Rq[3] = 2.0 * (qx * qy + qw * qz);
    Rq[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
    Rq[5] = 2.0 * (qy * qz - qw * qx);
    Rq[6] = 2.0 * (qx * qz - qw * qy);
    Rq[7] = 2.0 * (qy * qz + qw * qx);
    Rq[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
    const double s[3] = {exp(double(lf.x)), exp(double(lf.y)), exp(double(lf.z))};
    double M[9], Sig[9], W[9], Sc[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) M[3 * r + c] = Rq[3 * r + c] * s[c];
    // symmetric products are formed once per unordered pair (round 2)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = r; c < 3; ++c)
        Sig[3 * r + c] = Sig[3 * c + r] = M[3 * r] * M[3 * c] + M[3 * r + 1] * M[3 * c + 1] + M[3 * r + 2] * M[3 * c + 2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) W[3 * r + c] = R[3 * r] * Sig[c] + R[3 * r + 1] * Sig[3 + c] + R[3 * r + 2] * Sig[6 + c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = r; c < 3; ++c)
        Sc[3 * r + c] = Sc[3 * c + r] = W[3 * r] * R[3 * c] + W[3 * r + 1] * R[3 * c + 1] + W[3 * r + 2] * R[3 * c + 2];
    const double fx = a.fx, fy = a.fy;
    const double iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    const double J0 = fx * iz, J2 = -fx * x * iz2, J4 = fy * iz, J5 = -fy * y * iz2;
    // conic -> Sigma^I: G_S2 = -Conic G_M Conic, G_M = [[gA, gB/2], [gB/2, gC]]
    const double A = cn.x, B = cn.y, C = cn.z;
    const double hB = 0.5 * gB;
    const double t00 = A * gA + B * hB, t01 = A * hB + B * gC, t10 = B * gA + C * hB, t11 = B * hB + C * gC;
    const double S00 = -(t00 * A + t01 * B), S01 = -(t00 * B + t01 * C), S11 = -(t10 * B + t11 * C);
    // Sigma^I = J Sigma_c J^T: G_Sc = J^T G_S2 J, G_J = 2 G_S2 J Sigma_c, J = [[J0, 0, J2], [0, J4, J5]]
    // G_Sc = J^T G_S2 J written out (the structural zeros of J dropped)
    const double GS2[4] = {S00, S01, S01, S11};
    double GJ0[6], GJ[6];  // G_S2 J
    GJ0[0] = S00 * J0;
    GJ0[1] = S01 * J4;
    GJ0[2] = S00 * J2 + S01 * J5;
    GJ0[3] = S01 * J0;
    GJ0[4] = S11 * J4;
    GJ0[5] = S01 * J2 + S11 * J5;
    double GSc[9];
    GSc[0] = J0 * GJ0[0];
    GSc[1] = GSc[3] = J0 * GJ0[1];
    GSc[2] = GSc[6] = J0 * GJ0[2];
    GSc[4] = J4 * GJ0[4];
    GSc[5] = GSc[7] = J4 * GJ0[5];
    GSc[8] = J2 * GJ0[2] + J5 * GJ0[5];
    (void)GS2;
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        GJ[3 * r + c] = 2.0 * (GJ0[3 * r] * Sc[c] + GJ0[3 * r + 1] * Sc[3 + c] + GJ0[3 * r + 2] * Sc[6 + c]);
    // camera-frame mean p: through (u, v) (Eq. 1), J(p) and the depth term (Eq. 6)
    double gp[3];
    gp[0] = gu * fx * iz - GJ[2] * fx * iz2;
    gp[1] = gv * fy * iz - GJ[5] * fy * iz2;
    gp[2] = -gu * fx * x * iz2 - gv * fy * y * iz2 + gz - GJ[0] * fx * iz2 + GJ[2] * 2.0 * fx * x * iz3 -
            GJ[4] * fy * iz2 + GJ[5] * 2.0 * fy * y * iz3;
    if (kParams) {
      double gmu[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) gmu[c] = R[c] * gp[0] + R[3 + c] * gp[1] + R[6 + c] * gp[2];
      // G_Sigma = R^T G_Sc R; G_M = 2 G_Sigma M
      double tmp[9], GSig[9], GM3[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) tmp[3 * r + c] = R[r] * GSc[c] + R[3 + r] * GSc[3 + c] + R[6 + r] * GSc[6 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = r; c < 3; ++c)
          GSig[3 * r + c] = GSig[3 * c + r] = tmp[3 * r] * R[c] + tmp[3 * r + 1] * R[3 + c] + tmp[3 * r + 2] * R[6 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          GM3[3 * r + c] = 2.0 * (GSig[3 * r] * M[c] + GSig[3 * r + 1] * M[3 + c] + GSig[3 * r + 2] * M[6 + c]);
      double gls[3], GRq[9];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        gls[k] = s[k] * (GM3[k] * Rq[k] + GM3[3 + k] * Rq[3 + k] + GM3[6 + k] * Rq[6 + k]);
#pragma unroll
        for (int r = 0; r < 3; ++r) GRq[3 * r + k] = GM3[3 * r + k] * s[k];
      }
      // dR(q^)/dq^ contracted with G_Rq
      const double gw = 2.0 * (-qz * GRq[1] + qy * GRq[2] + qz * GRq[3] - qx * GRq[5] - qy * GRq[6] + qx * GRq[7]);
      const double gx = 2.0 * (qy * GRq[1] + qz * GRq[2] + qy * GRq[3] - 2.0 * qx * GRq[4] - qw * GRq[5] + qz * GRq[6] +
                               qw * GRq[7] - 2.0 * qx * GRq[8]);
      const double gy = 2.0 * (-2.0 * qy * GRq[0] + qx * GRq[1] + qw * GRq[2] + qx * GRq[3] + qz * GRq[5] - qw * GRq[6] +
                               qz * GRq[7] - 2.0 * qy * GRq[8]);
      const double gzq = 2.0 * (-2.0 * qz * GRq[0] - qw * GRq[1] + qx * GRq[2] + qw * GRq[3] - 2.0 * qz * GRq[4] +
                                qy * GRq[5] + qx * GRq[6] + qy * GRq[7]);
      const double dot = gw * qw + gx * qx + gy * qy + gzq * qz;
      // q^ = q / |q| (R18)
      if (a.atomic_acc) {
        red_add_v4(reinterpret_cast<float *>(a.g_mean_opa + i), float(gmu[0]), float(gmu[1]), float(gmu[2]), gb.z);
        red_add_v4(reinterpret_cast<float *>(a.g_quat + i), float((gw - qw * dot) * iq), float((gx - qx * dot) * iq),
                   float((gy - qy * dot) * iq), float((gzq - qz * dot) * iq));
        red_add_v4(reinterpret_cast<float *>(a.g_logscale + i), float(gls[0]), float(gls[1]), float(gls[2]), 0.f);
        red_add_v4(reinterpret_cast<float *>(a.g_rgb + i), gc.x, gc.y, gc.z, 0.f);
      } else {
        a.g_mean_opa[i] = make_float4(float(old_m.x + gmu[0]), float(old_m.y + gmu[1]), float(old_m.z + gmu[2]),
                                      old_m.w + gb.z);
        a.g_quat[i] = make_float4(float(old_q.x + (gw - qw * dot) * iq), float(old_q.y + (gx - qx * dot) * iq),
                                  float(old_q.z + (gy - qy * dot) * iq), float(old_q.w + (gzq - qz * dot) * iq));
        a.g_logscale[i] = make_float4(float(old_l.x + gls[0]), float(old_l.y + gls[1]), float(old_l.z + gls[2]), old_l.w);
        a.g_rgb[i] = make_float4(old_c.x + gc.x, old_c.y + gc.y, old_c.z + gc.z, old_c.w);
      }
    }
    if (kPose) {
      // dL/dt = dL/dp; dL/dR = dL/dp mu^T + 2 G_Sc R Sigma
      const double *RS = W;  // R Sigma
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          pose[3 * r + c] =
              float(gp[r] * mu[c] + 2.0 * (GSc[3 * r] * RS[c] + GSc[3 * r + 1] * RS[3 + c] + GSc[3 * r + 2] * RS[6 + c]));
#pragma unroll
      for (int k = 0; k < 3; ++k) pose[9 + k] = float(gp[k]);
    }
  }
  if (kPose) {
    // fixed-order block reduction: warp shuffles, then warp partials summed by thread order
    __shared__ float sh[kGaussThreads / 32][12];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      float v = pose[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 12) {
      float v = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sh[w][threadIdx.x];
      a.pose_partials[size_t(blockIdx.x) * 12 + threadIdx.x] = v;
    }
  }
}

}  // namespace gs

extern "C" size_t gs_bwd_workspace_bytes(int32_t n) {
  if (n < 0) return 0;
  return size_t(n > 0 ? n : 1) * gs::kG2 * sizeof(float);
}

extern "C" int32_t gs_pose_partials_count(int32_t n) {
  if (n < 0) return 0;
  return n > 0 ? (n + gs::kGaussThreads - 1) / gs::kGaussThreads : 1;
}

extern "C" int gs_render_bwd(gs_params p, const gs_view *view, gs_camera cam, gs_proj pr, const int32_t *sorted_idx,
                             const int32_t *tile_range, const int32_t *tile_order, const float *T_final, const int32_t *n_contrib,
                             const float *dL_dcolor, const float *dL_ddepth, const float *dL_dalpha, uint32_t flags,
                             void *ws, size_t ws_bytes, float *g_mean_opa, float *g_quat, float *g_logscale,
                             float *g_rgb, float *pose_partials, uint32_t *tile_done, void *stream) {
  using namespace gs;
  const bool want_params = flags & GS_GRAD_PARAMS, want_pose = flags & GS_GRAD_POSE;
  const bool run_pixels = !(flags & GS_BWD_GAUSS_ONLY), run_gauss = !(flags & GS_BWD_PIXELS_ONLY);
  if (p.n < 0 || !view || !camera_ok(cam) || !tile_range || !T_final || !n_contrib || !dL_dcolor || !dL_ddepth ||
      (flags & ~(GS_GRAD_PARAMS | GS_GRAD_POSE | GS_BWD_PIXELS_ONLY | GS_BWD_GAUSS_ONLY | GS_BWD_ATOMIC_ACC)) ||
      !(want_params || want_pose) || !(run_pixels || run_gauss)) {
    set_error("gs_render_bwd: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (want_params && (!g_mean_opa || !g_quat || !g_logscale || !g_rgb || !aligned16(g_mean_opa) ||
                      !aligned16(g_quat) || !aligned16(g_logscale) || !aligned16(g_rgb))) {
    set_error("gs_render_bwd: GS_GRAD_PARAMS needs four aligned gradient arrays");
    return GS_ERR_INVALID_ARG;
  }
  if (want_pose && !pose_partials) {
    set_error("gs_render_bwd: GS_GRAD_POSE needs pose_partials");
    return GS_ERR_INVALID_ARG;
  }
  if (p.n > 0) {
    const void *ptrs[] = {p.mean_opa, p.quat, p.logscale, pr.uv, pr.coef, pr.rgbz, pr.conic_o};
    for (const void *x : ptrs)
      if (!x || !aligned16(x)) {
        set_error("gs_render_bwd: null or misaligned parameter/projection array");
        return GS_ERR_INVALID_ARG;
      }
    if (!pr.tiles_touched) {
      set_error("gs_render_bwd: null tiles_touched");
      return GS_ERR_INVALID_ARG;
    }
  }
  if (!ws || ws_bytes < gs_bwd_workspace_bytes(p.n) || !aligned16(ws)) {
    set_error("gs_render_bwd: workspace too small or misaligned");
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  float *grad2d = static_cast<float *>(ws);
  if (p.n == 0) return GS_OK;
  BwdArgs b{reinterpret_cast<const double2 *>(pr.uv), reinterpret_cast<const float4 *>(pr.coef),
            reinterpret_cast<const float4 *>(pr.rgbz), reinterpret_cast<const float4 *>(pr.conic_o), sorted_idx,
            reinterpret_cast<const int2 *>(tile_range), tile_order, T_final, n_contrib, dL_dcolor, dL_ddepth, dL_dalpha,
            cam.width, cam.height, tiles_x(cam), grad2d, tile_done, tiles_x(cam) * tiles_y(cam), p.n};
  const int T = tiles_x(cam) * tiles_y(cam);
  if (run_pixels) {
    void (*kern)(BwdArgs) = want_params ? (dL_dalpha ? k_bwd_pixels<true, true> : k_bwd_pixels<true, false>)
                                        : (dL_dalpha ? k_bwd_pixels<false, true> : k_bwd_pixels<false, false>);
    // programmatic dependent launch (with tile_done: overlaps the forward's
    // tail tile by tile)
    launch_pdl(kern, dim3(T), dim3(BG::kThreads), 0, s, b);
  }
  if (!run_gauss) return check_launch("gs_render_bwd");
  GaussArgs g{p, view, cam.fx, cam.fy, reinterpret_cast<const float4 *>(pr.conic_o), pr.tiles_touched, grad2d,
              reinterpret_cast<float4 *>(g_mean_opa), reinterpret_cast<float4 *>(g_quat),
              reinterpret_cast<float4 *>(g_logscale), reinterpret_cast<float4 *>(g_rgb), pose_partials,
              (flags & GS_BWD_ATOMIC_ACC) != 0};
  const int blocks = gs_pose_partials_count(p.n);
  if (want_params && want_pose)
    launch_pdl(k_bwd_gauss<true, true>, dim3(blocks), dim3(kGaussThreads), 0, s, g);
  else if (want_params)
    launch_pdl(k_bwd_gauss<true, false>, dim3(blocks), dim3(kGaussThreads), 0, s, g);
  else
    launch_pdl(k_bwd_gauss<false, true>, dim3(blocks), dim3(kGaussThreads), 0, s, g);
  return check_launch("gs_render_bwd");
}


