// render_fwd.cu — S3 gs_render_fwd: per-tile front-to-back alpha compositing
// of colour (Eq. 3), depth (Eq. 6) and accumulated alpha (P:133-141,
// P:161-166; R11-R15).
//
// One CTA (4 warps) per 16x16 tile; each warp owns an 8x8 pixel block and
// each thread 2 adjacent pixels of a row (raster_common.cuh).  The tile's
// depth-ordered list is staged in batches of 128 records in shared memory
// (each thread gathers one: uv in fp64 -> tile-local fp32 offsets (H2), the
// H2b entry terms, rgb and camera depth, plus the set of warp blocks met by a
// conservative box of the entry's alpha >= 1/255 region).  Every warp then
// compacts the indices of the entries that meet its block into a hit list and
// walks it: the row terms of the exponent are computed once per (thread,
// entry) and the 2 pixels are evaluated as one fp32x2 pair (FFMA2); ex2 and
// the branch-free blend (also FFMA2) run only for entries that pass the
// exponent pre-test at some pixel of the warp.  The CTA leaves as soon as all
// of its pixels have terminated (T < 1e-4).
#include "raster_common.cuh"

namespace gs {

struct FwdArgs {
  const double2 *uv;
  const float4 *coef;
  const float4 *rgbz;
  const int32_t *sorted_idx;
  const int2 *tile_range;
  const int32_t *tile_order;
  int W, H, TX;
  float *color, *depth, *alpha, *T_final;
  int32_t *n_contrib, *stats, *tile_work;
  // fused L1 gradient epilogue (gs_render_fwd_l1): targets, device scales
  // (lambda_c / 3HW, lambda_d / |V|, |V|) from gs_loss_scales, gradient maps,
  // per-tile fp64 sums of |C - C*| and of |D - D*| over valid pixels (nullable)
  const float *tc, *td, *scales;
  float *gC, *gD;
  double *loss_part;
  // per-tile completion flags for a programmatically dependent backward
  // (gs_render_bwd with the same tile_done); nullable
  uint32_t *tile_done;
};

#ifndef FWD_NP
#define FWD_NP 1
#endif
#ifndef FWD_WX
#define FWD_WX 8
#endif
// Forward geometry: NP fp32x2 pixel pairs per thread on WX-wide warp blocks.
//   NP = 1, WX = 8:  4 warps on 8x8 blocks, 2 px / thread
//   NP = 2, WX = 16: 2 warps on 16x8 strips, 4 px / thread
// resident CTAs per SM the register budget must allow: 8 (64 registers, no
// spills; 72 without the cap = 7 CTAs): 94.2 -> 91.0 µs alone, 2816 it/s;
// 9 no change, 10 (48 registers) 106 µs
#ifndef FWD_PDL
#define FWD_PDL 1
#endif
#ifndef FWD_MINB
#define FWD_MINB 8
#endif
constexpr int kFNP = FWD_NP;
constexpr int kFWX = FWD_WX;
using FG = Geo<2 * kFNP, kFWX>;

// per-thread compositing state of one pixel pair
struct FwdPix {
  float2 T, c0, c1, c2, D, A;
  int last0, last1, ncon0, ncon1, term0, term1;
};

// One list entry at a pixel pair: alpha decision (R11) and the blend of
// Eqs. 3, 6 and R14, branch-free (alpha = 0 leaves the state bit-identical).
template <bool kStats>
__device__ __forceinline__ void fwd_blend(FwdPix &s, float2 e, bool q0, bool q1, float4 c, int pos) {
  // q: live and alpha~ >= 1/255 (e >= kExpMin, R2'); a skipped pixel's
  // exponent becomes -inf, so alpha = 2^-inf = 0 (R11)
  const float a0 = fminf(ex2_approx(q0 ? e.x : -INFINITY), kAlphaMax);
  const float a1 = fminf(ex2_approx(q1 ? e.y : -INFINITY), kAlphaMax);
  s.last0 = q0 ? pos : s.last0;
  s.last1 = q1 ? pos : s.last1;
  const float2 wt = __fmul2_rn(make_float2(a0, a1), s.T);           // alpha_j T_j
  s.c0 = __ffma2_rn(make_float2(c.x, c.x), wt, s.c0);               // Eq. 3
  s.c1 = __ffma2_rn(make_float2(c.y, c.y), wt, s.c1);
  s.c2 = __ffma2_rn(make_float2(c.z, c.z), wt, s.c2);
  s.D = __ffma2_rn(make_float2(c.w, c.w), wt, s.D);                 // Eq. 6 (camera-frame z, R12)
  s.A = __fadd2_rn(s.A, wt);                                        // R14
  s.T = __ffma2_rn(make_float2(-a0, -a1), s.T, s.T);                // T_{j+1} = T_j (1 - alpha_j)
  if (kStats) {
    s.ncon0 += q0;
    s.ncon1 += q1;
    s.term0 = (q0 && !(s.T.x >= kTEps)) ? pos : s.term0;  // include, then stop (R11)
    s.term1 = (q1 && !(s.T.y >= kTEps)) ? pos : s.term1;
  }
}

// one staged list entry of the forward
struct __align__(16) FwdRec {
  float4 p;     // entry terms (a', b', d', K)
  float4 rgbz;  // colour, camera depth
  float2 q;     // (DV, log2 o)
  float2 pad;
};

__device__ __forceinline__ bool any_live(const FwdPix s[kFNP]) {
  bool l = false;
#pragma unroll
  for (int h = 0; h < kFNP; ++h) l |= s[h].T.x >= kTEps || s[h].T.y >= kTEps;
  return l;
}

// one hit at all of the thread's pairs: returns the pass test, blends if any lane passes
template <bool kStats>
__device__ __forceinline__ void fwd_entry(FwdPix s[kFNP], const float2 e[kFNP], const FwdRec &rc, int pos) {
  bool p[kFNP][2], any = false;
#pragma unroll
  for (int h = 0; h < kFNP; ++h) {
    // live (T >= 1e-4, compared where it is used: no flag to keep) and
    // alpha~ >= 1/255
    p[h][0] = s[h].T.x >= kTEps && e[h].x >= kExpMin;
    p[h][1] = s[h].T.y >= kTEps && e[h].y >= kExpMin;
    any |= p[h][0] || p[h][1];
  }
  if (!__any_sync(0xffffffffu, any)) return;
  const float4 c = rc.rgbz;
#pragma unroll
  for (int h = 0; h < kFNP; ++h) fwd_blend<kStats>(s[h], e[h], p[h][0], p[h][1], c, pos);
}

template <bool kStats, bool kL1 = false>
__global__ void __launch_bounds__(FG::kThreads, FWD_MINB) k_render_fwd(FwdArgs a) {
  // one staged record per entry; record kBatch is a sentinel entry whose exponent is -inf
  __shared__ FwdRec s_rec[kBatch + 1];
  __shared__ unsigned char s_mask[kBatch];
  __shared__ unsigned char s_list[FG::kWarps][kBatch + 2];
  // wait for the predecessor grid BEFORE reading any of its outputs (the
  // launch order is written by the last kernel of gs_bin_sort); then the
  // dependent backward of gs_render_fwd_l1(tile_done) may launch
  pdl_begin();
  const int tile = a.tile_order ? __ldg(a.tile_order + blockIdx.x) : int(blockIdx.x);
  GS_ASSERT(tile >= 0 && tile < int(gridDim.x));
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int w = threadIdx.x >> 5;
  const PixGeom pg = pix_geom<FG>(tx, ty, a.H);
  const double ox = double(tx * kTile), oy = double(ty * kTile);
  const int2 range = a.tile_range[tile];
  GS_ASSERT(range.x >= 0 && range.x <= range.y);
  float2 fx[kFNP];
#pragma unroll
  for (int h = 0; h < kFNP; ++h) fx[h] = make_float2(pg.fpx0 + 2.f * h, pg.fpx0 + 2.f * h + 1.f);
  if (threadIdx.x == 0) {
    s_rec[kBatch].p = make_float4(0.f, 0.f, 0.f, 0.f);
    s_rec[kBatch].q = make_float2(0.f, -INFINITY);
  }
  // a pixel composites while T >= 1e-4 (include, then stop: T < 1e-4 happens
  // exactly at the stopping entry); pixels outside the image start with T = 0
  FwdPix s[kFNP];
#pragma unroll
  for (int h = 0; h < kFNP; ++h) {
    s[h].T = make_float2((pg.row_in && pg.px0 + 2 * h < a.W) ? 1.f : 0.f,
                         (pg.row_in && pg.px0 + 2 * h + 1 < a.W) ? 1.f : 0.f);
    s[h].c0 = s[h].c1 = s[h].c2 = s[h].D = s[h].A = make_float2(0.f, 0.f);
    s[h].last0 = s[h].last1 = s[h].ncon0 = s[h].ncon1 = 0;
    s[h].term0 = s[h].term1 = range.y - range.x;  // entries scanned if the pixel never terminates
  }
  for (int start = range.x; start < range.y; start += kBatch) {
    if (__syncthreads_count(any_live(s)) == 0) break;
#pragma unroll
    for (int r = 0; r < FG::kRecPerThread; ++r) {
      const int i = r * FG::kThreads + threadIdx.x;
      const int k = start + i;
      if (k < range.y) {
        const int g = __ldg(a.sorted_idx + k);
        GS_ASSERT(g >= 0);
        const double2 u = __ldg(a.uv + g);
        const float4 cf = __ldg(a.coef + g);
        const float ul = float(u.x - ox), vl = float(u.y - oy);
        const EntryTerms et = entry_terms(cf, ul, vl);
        FwdRec &rc = s_rec[i];
        rc.p = et.p;
        rc.q = et.q;
        rc.rgbz = __ldg(a.rgbz + g);
        s_mask[i] = (unsigned char)entry_block_mask<FG>(cf, ul, vl);
      }
    }
    __syncthreads();
    // walk this warp's hits in list order, two per step (their exponents are
    // independent; the blends stay in order).  Entries that miss the warp's
    // block cannot pass the exponent pre-test at any of its pixels (no
    // decision changes); list[nh] is the sentinel.
    unsigned char *list = s_list[w];
    const int nh = warp_hit_list(s_mask, min(kBatch, range.y - start), list, kBatch);
    const int base = start - range.x + 1;
    // the warp's early exit is tested once per 32 hits (outer loop), not per step
    for (int k0 = 0; k0 < nh; k0 += 32) {
      if (!__any_sync(0xffffffffu, any_live(s))) break;
      const int k1 = min(nh, k0 + 32);
      for (int k = k0; k < k1; k += 2) {
        const int ja = list[k], jb = list[k + 1];
        const RowTerms ra = row_terms(s_rec[ja].p, s_rec[ja].q, pg.fpy);
        const RowTerms rb = row_terms(s_rec[jb].p, s_rec[jb].q, pg.fpy);
        float2 ea[kFNP], eb[kFNP];
#pragma unroll
        for (int h = 0; h < kFNP; ++h) {
          ea[h] = pair_exponent(ra, fx[h]);
          eb[h] = pair_exponent(rb, fx[h]);
        }
        fwd_entry<kStats>(s, ea, s_rec[ja], base + ja);
        fwd_entry<kStats>(s, eb, s_rec[jb], base + jb);
      }
    }
  }
  if (a.tile_work) {
    // the backward's work on this tile: its two warps each walk a 16x8 strip
    // back from the strip's LARGEST n_contrib (SIMT) and the CTA lasts as long
    // as its slower warp, so the proxy is the larger of the two strips' maximum
    // n_contrib (a sum over pixels ranks a tile with a few deep pixels too low
    // in gs_tile_order's heaviest-first order: measured 199 -> 172 us for the
    // backward, TW_MAX=0 is the sum of the two strip maxima: 186 us)
    __shared__ int s_strip[2], s_work;
    if (threadIdx.x < 2) s_strip[threadIdx.x] = 0;
    __syncthreads();
    int wk = 0;
#pragma unroll
    for (int h = 0; h < kFNP; ++h) wk = max(wk, max(s[h].last0, s[h].last1));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wk = max(wk, __shfl_xor_sync(0xffffffffu, wk, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&s_strip[min(1, (FG::by(w) * 2) / kTile)], wk);
    __syncthreads();
#ifndef TW_MAX
#define TW_MAX 1
#endif
    if (threadIdx.x == 0) s_work = TW_MAX ? max(s_strip[0], s_strip[1]) : s_strip[0] + s_strip[1];
    __syncthreads();
    if (threadIdx.x == 0) a.tile_work[tile] = s_work;
  }
  const size_t HW = size_t(a.W) * a.H;
  double l1c = 0.0, l1d = 0.0;  // this thread's |residual| sums (kL1)
#pragma unroll
  for (int h = 0; h < kFNP; ++h) {
    if (!pg.row_in) break;
    const float cc0[2] = {s[h].c0.x, s[h].c0.y}, cc1[2] = {s[h].c1.x, s[h].c1.y}, cc2[2] = {s[h].c2.x, s[h].c2.y},
                DD[2] = {s[h].D.x, s[h].D.y}, AA[2] = {s[h].A.x, s[h].A.y}, TT[2] = {s[h].T.x, s[h].T.y};
    const int ll[2] = {s[h].last0, s[h].last1}, nc[2] = {s[h].ncon0, s[h].ncon1}, tm[2] = {s[h].term0, s[h].term1};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (pg.px0 + 2 * h + k >= a.W) break;
      const size_t q = size_t(pg.py) * a.W + pg.px0 + 2 * h + k;
      a.color[q] = cc0[k];
      a.color[HW + q] = cc1[k];
      a.color[2 * HW + q] = cc2[k];
      a.depth[q] = DD[k];
      a.alpha[q] = AA[k];
      a.T_final[q] = TT[k];
      a.n_contrib[q] = ll[k];
      if (kStats) {
        a.stats[q] = tm[k];  // entries scanned = termination position or list length
        a.stats[HW + q] = nc[k];
      }
      if (kL1) {  // gs_loss's gradient maps, the same fp32 values (weight 1, sign(0) = 0, R21)
        const float sc = __ldg(a.scales), sd = __ldg(a.scales + 1);
        const float cc[3] = {cc0[k], cc1[k], cc2[k]};
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float r = cc[ch] - __ldg(a.tc + ch * HW + q);
          a.gC[ch * HW + q] = sc * 1.f * float((r > 0.f) - (r < 0.f));
          l1c += fabs(double(r));
        }
        const float t = __ldg(a.td + q);
        const float r = DD[k] - t;
        a.gD[q] = t > 0.f ? sd * 1.f * float((r > 0.f) - (r < 0.f)) : 0.f;
        if (t > 0.f) l1d += fabs(double(r));
      }
    }
  }
  if (kL1 && a.loss_part) {  // the tile's sums, fixed order: warp shuffles, then warps in order
    __shared__ double s_l1[FG::kWarps][2];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l1c += __shfl_xor_sync(0xffffffffu, l1c, o);
      l1d += __shfl_xor_sync(0xffffffffu, l1d, o);
    }
    if ((threadIdx.x & 31) == 0) {
      s_l1[w][0] = l1c;
      s_l1[w][1] = l1d;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double c = 0.0, d = 0.0;
      for (int k = 0; k < FG::kWarps; ++k) {
        c += s_l1[k][0];
        d += s_l1[k][1];
      }
      a.loss_part[2 * size_t(tile)] = c;
      a.loss_part[2 * size_t(tile) + 1] = d;
    }
  }
  if (kL1 && a.tile_done) {  // this tile's outputs are complete: release its flag
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.tile_done + tile), "r"(1u) : "memory");
  }
}

}  // namespace gs

extern "C" int gs_render_fwd(gs_proj pr, const int32_t *sorted_idx, const int32_t *tile_range,
                             const int32_t *tile_order, gs_camera cam, float *color, float *depth, float *alpha,
                             float *T_final, int32_t *n_contrib, int32_t *stats, int32_t *tile_work, void *stream) {
  using namespace gs;
  if (!camera_ok(cam) || !tile_range || !color || !depth || !alpha || !T_final || !n_contrib) {
    set_error("gs_render_fwd: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (!pr.uv || !pr.coef || !pr.rgbz || !aligned16(pr.uv) || !aligned16(pr.coef) || !aligned16(pr.rgbz) ||
      (reinterpret_cast<uintptr_t>(tile_range) & 7u)) {
    set_error("gs_render_fwd: null or misaligned projection arrays");
    return GS_ERR_INVALID_ARG;
  }
  FwdArgs a{reinterpret_cast<const double2 *>(pr.uv), reinterpret_cast<const float4 *>(pr.coef),
            reinterpret_cast<const float4 *>(pr.rgbz), sorted_idx, reinterpret_cast<const int2 *>(tile_range),
            tile_order, cam.width, cam.height, tiles_x(cam), color, depth, alpha, T_final, n_contrib, stats,
            tile_work, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  const int T = tiles_x(cam) * tiles_y(cam);
  if (stats)
    launch_pdl(k_render_fwd<true>, dim3(T), dim3(FG::kThreads), 0, as_stream(stream), a);
  else
    launch_pdl(k_render_fwd<false>, dim3(T), dim3(FG::kThreads), 0, as_stream(stream), a);
  return check_launch("gs_render_fwd");
}

extern "C" int gs_render_fwd_l1(gs_proj pr, const int32_t *sorted_idx, const int32_t *tile_range,
                                const int32_t *tile_order, gs_camera cam, float *color, float *depth, float *alpha,
                                float *T_final, int32_t *n_contrib, int32_t *tile_work, const float *tgt_color,
                                const float *tgt_depth, const float *scales, float *dL_dcolor, float *dL_ddepth,
                                double *loss_part, uint32_t *tile_done, void *stream) {
  using namespace gs;
  if (!camera_ok(cam) || !tile_range || !color || !depth || !alpha || !T_final || !n_contrib || !tgt_color ||
      !tgt_depth || !scales || !dL_dcolor || !dL_ddepth) {
    set_error("gs_render_fwd_l1: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (!pr.uv || !pr.coef || !pr.rgbz || !aligned16(pr.uv) || !aligned16(pr.coef) || !aligned16(pr.rgbz) ||
      (reinterpret_cast<uintptr_t>(tile_range) & 7u)) {
    set_error("gs_render_fwd_l1: null or misaligned projection arrays");
    return GS_ERR_INVALID_ARG;
  }
  FwdArgs a{reinterpret_cast<const double2 *>(pr.uv), reinterpret_cast<const float4 *>(pr.coef),
            reinterpret_cast<const float4 *>(pr.rgbz), sorted_idx, reinterpret_cast<const int2 *>(tile_range),
            tile_order, cam.width, cam.height, tiles_x(cam), color, depth, alpha, T_final, n_contrib, nullptr,
            tile_work, tgt_color, tgt_depth, scales, dL_dcolor, dL_ddepth, loss_part, tile_done};
  const int T = tiles_x(cam) * tiles_y(cam);
  launch_pdl_if(FWD_PDL, k_render_fwd<false, true>, dim3(T), dim3(FG::kThreads), 0, as_stream(stream), a);
  return check_launch("gs_render_fwd_l1");
}
