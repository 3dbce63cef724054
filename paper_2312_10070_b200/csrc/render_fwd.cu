// render_fwd.cu — S3 gs_render_fwd: per-tile front-to-back alpha compositing
// of colour (Eq. 3), depth (Eq. 6) and accumulated alpha (P:133-141,
// P:161-166; R11-R15).
//
// One CTA (4 warps) per 16x16 tile; each thread owns 2 pixels of a row
// (raster_common.cuh).  The tile's depth-ordered list is staged in batches of
// 128 records in shared memory (each thread gathers one: uv in fp64 ->
// tile-local fp32 offsets (H2), the H2b coefficients, rgb and camera depth,
// plus a conservative box of the entry's alpha >= 1/255 region).  A warp
// skips entries whose box misses its 16x4 strip; otherwise the row terms of
// the exponent are computed once per (thread, entry) and reused by the 2
// pixels (2 FFMA + compare per pixel); ex2 and the blend run only for entries
// that pass the exponent pre-test.  The CTA leaves as soon as all of its
// pixels have terminated (T < 1e-4).
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
};

constexpr int kFPX = 2;  // pixels per thread in the forward
using FG = Geo<kFPX>;

template <bool kStats>
__global__ void __launch_bounds__(FG::kThreads) k_render_fwd(FwdArgs a) {
  __shared__ float2 s_uv[kBatch];
  __shared__ float4 s_coef[kBatch];
  __shared__ float4 s_rgbz[kBatch];
  __shared__ unsigned char s_mask[kBatch];
  const int tile = a.tile_order ? __ldg(a.tile_order + blockIdx.x) : int(blockIdx.x);
  const int tx = tile % a.TX, ty = tile / a.TX;
  const PixGeom pg = pix_geom<kFPX>(tx, ty, a.H);
  const double ox = double(tx * kTile), oy = double(ty * kTile);
  const int2 range = a.tile_range[tile];
  float T[kFPX], c0[kFPX], c1[kFPX], c2[kFPX], D[kFPX], A[kFPX];
  // a pixel composites while T >= 1e-4 (include, then stop: T < 1e-4 happens
  // exactly at the stopping entry); pixels outside the image start with T = 0
  int last[kFPX], ncon[kFPX], term[kFPX];
#pragma unroll
  for (int k = 0; k < kFPX; ++k) {
    T[k] = (pg.row_in && pg.px0 + k < a.W) ? 1.f : 0.f;
    c0[k] = c1[k] = c2[k] = D[k] = A[k] = 0.f;
    last[k] = ncon[k] = 0;
    term[k] = range.y - range.x;  // entries scanned if the pixel never terminates
  }
  for (int start = range.x; start < range.y; start += kBatch) {
    if (__syncthreads_count(T[0] >= kTEps || T[1] >= kTEps) == 0) break;
    static_assert(FG::kRecPerThread == 1, "one staged record per thread");
    {
      const int k = start + threadIdx.x;
      if (k < range.y) {
        const int g = __ldg(a.sorted_idx + k);
        const double2 u = __ldg(a.uv + g);
        const float4 cf = __ldg(a.coef + g);
        const float ul = float(u.x - ox), vl = float(u.y - oy);
        s_uv[threadIdx.x] = make_float2(ul, vl);
        s_coef[threadIdx.x] = cf;
        s_rgbz[threadIdx.x] = __ldg(a.rgbz + g);
        s_mask[threadIdx.x] = (unsigned char)box_strip_mask<kFPX>(entry_box(cf, ul, vl));
      }
    }
    __syncthreads();
    unsigned hits[kBatch / 32];
    warp_hits(s_mask, min(kBatch, range.y - start), hits);
    // walk this warp's hits in list order; entries that miss its strip cannot
    // pass the exponent pre-test at any of its pixels (no decision changes).
    // The blend is branch-free: a pixel that does not composite uses alpha = 0,
    // which leaves C, D, A and T bit-identical.
#pragma unroll
    for (int h = 0; h < kBatch / 32; ++h) {
      unsigned bits = hits[h];
      if (bits && !__any_sync(0xffffffffu, T[0] >= kTEps || T[1] >= kTEps)) break;
      while (bits) {
        const int j = h * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
        const float2 ul = s_uv[j];
        const RowTerms rt = row_terms(s_coef[j], ul.x, ul.y, pg.fpy);
        float e[kFPX];
        bool pass[kFPX];
#pragma unroll
        for (int k = 0; k < kFPX; ++k) {
          e[k] = pixel_exponent(rt, pg.fpx0 + float(k));
          pass[k] = e[k] >= kExpSkip && T[k] >= kTEps;
        }
        if (!__any_sync(0xffffffffu, pass[0] || pass[1])) continue;
        const float4 c = s_rgbz[j];
        const int pos = start - range.x + j + 1;
#pragma unroll
        for (int k = 0; k < kFPX; ++k) {
          float al = fminf(ex2_approx(e[k]), kAlphaMax);
          al = (pass[k] && al >= kAlphaMin) ? al : 0.f;  // skip (R11)
          const float w = __fmul_rn(al, T[k]);           // alpha_j T_j
          c0[k] = __fmaf_rn(c.x, w, c0[k]);              // Eq. 3
          c1[k] = __fmaf_rn(c.y, w, c1[k]);
          c2[k] = __fmaf_rn(c.z, w, c2[k]);
          D[k] = __fmaf_rn(c.w, w, D[k]);                // Eq. 6 (camera-frame z, R12)
          A[k] = __fadd_rn(A[k], w);                     // R14
          T[k] = __fmul_rn(T[k], __fsub_rn(1.f, al));
          last[k] = al > 0.f ? pos : last[k];
          if (kStats) {
            ncon[k] += al > 0.f;
            term[k] = (al > 0.f && T[k] < kTEps) ? pos : term[k];  // include, then stop (R11)
          }
        }
      }
    }
  }
  if (a.tile_work) {  // the backward's work on this tile: sum of n_contrib
    __shared__ int s_work;
    if (threadIdx.x == 0) s_work = 0;
    __syncthreads();
    int wk = last[0] + last[1];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wk += __shfl_xor_sync(0xffffffffu, wk, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s_work, wk);
    __syncthreads();
    if (threadIdx.x == 0) a.tile_work[tile] = s_work;
  }
  if (!pg.row_in) return;
  const size_t HW = size_t(a.W) * a.H;
#pragma unroll
  for (int k = 0; k < kFPX; ++k) {
    if (pg.px0 + k >= a.W) break;
    const size_t q = size_t(pg.py) * a.W + pg.px0 + k;
    a.color[q] = c0[k];
    a.color[HW + q] = c1[k];
    a.color[2 * HW + q] = c2[k];
    a.depth[q] = D[k];
    a.alpha[q] = A[k];
    a.T_final[q] = T[k];
    a.n_contrib[q] = last[k];
    if (kStats) {
      a.stats[q] = term[k];  // entries scanned = termination position or list length
      a.stats[HW + q] = ncon[k];
    }
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
            tile_work};
  const int T = tiles_x(cam) * tiles_y(cam);
  if (stats)
    k_render_fwd<true><<<T, FG::kThreads, 0, as_stream(stream)>>>(a);
  else
    k_render_fwd<false><<<T, FG::kThreads, 0, as_stream(stream)>>>(a);
  return check_launch("gs_render_fwd");
}
