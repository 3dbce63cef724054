// render_fwd.cu — S3 gs_render_fwd: per-tile front-to-back alpha compositing
// of colour (Eq. 3), depth (Eq. 6) and accumulated alpha (P:133-141,
// P:161-166; R11-R15).
//
// One CTA per 16x16 tile, one pixel per thread.  The tile's depth-ordered
// list is staged in batches of 256 records in shared memory: each thread
// gathers one record (uv in fp64 -> tile-local fp32 offsets (H2), the H2b
// coefficients, rgb and camera depth).  Every thread then walks the batch;
// the CTA leaves as soon as all of its pixels have terminated (T < 1e-4).
#include "gs_internal.cuh"

namespace gs {

struct FwdArgs {
  const double2 *uv;
  const float4 *coef;
  const float4 *rgbz;
  const int32_t *sorted_idx;
  const int2 *tile_range;
  int W, H, TX;
  float *color, *depth, *alpha, *T_final;
  int32_t *n_contrib, *stats;
};

template <bool kStats>
__global__ void __launch_bounds__(kTilePx) k_render_fwd(FwdArgs a) {
  __shared__ float2 s_uv[kTilePx];
  __shared__ float4 s_coef[kTilePx];
  __shared__ float4 s_rgbz[kTilePx];
  const int tile = blockIdx.x;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x / kTile;
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < a.W && py < a.H;
  const double ox = double(tx * kTile), oy = double(ty * kTile);
  const float fpx = float(lx), fpy = float(ly);
  const int2 range = a.tile_range[tile];
  bool done = !inside;
  float T = 1.f, c0 = 0.f, c1 = 0.f, c2 = 0.f, D = 0.f, A = 0.f;
  int last = 0, nscan = 0, ncon = 0;
  for (int start = range.x; start < range.y; start += kTilePx) {
    if (__syncthreads_count(done) == kTilePx) break;
    const int k = start + threadIdx.x;
    if (k < range.y) {
      const int g = __ldg(a.sorted_idx + k);
      const double2 u = __ldg(a.uv + g);
      s_uv[threadIdx.x] = make_float2(float(u.x - ox), float(u.y - oy));
      s_coef[threadIdx.x] = __ldg(a.coef + g);
      s_rgbz[threadIdx.x] = __ldg(a.rgbz + g);
    }
    __syncthreads();
    const int cnt = min(kTilePx, range.y - start);
    if (!done) {
      for (int j = 0; j < cnt; ++j) {
        const float2 ul = s_uv[j];
        float dx, dy;
        const float e = alpha_exponent(s_coef[j], ul.x, ul.y, fpx, fpy, dx, dy);
        if (kStats) ++nscan;
        float al, at;
        if (!alpha_decide(e, al, at)) continue;
        const float4 c = s_rgbz[j];
        const float w = __fmul_rn(al, T);  // alpha_j T_j
        c0 = __fmaf_rn(c.x, w, c0);        // Eq. 3
        c1 = __fmaf_rn(c.y, w, c1);
        c2 = __fmaf_rn(c.z, w, c2);
        D = __fmaf_rn(c.w, w, D);          // Eq. 6 (camera-frame z, R12)
        A = __fadd_rn(A, w);               // R14
        T = __fmul_rn(T, __fsub_rn(1.f, al));
        last = start - range.x + j + 1;
        if (kStats) ++ncon;
        if (T < kTEps) {                   // include, then stop (R11)
          done = true;
          break;
        }
      }
    }
  }
  if (inside) {
    const size_t HW = size_t(a.W) * a.H, q = size_t(py) * a.W + px;
    a.color[q] = c0;
    a.color[HW + q] = c1;
    a.color[2 * HW + q] = c2;
    a.depth[q] = D;
    a.alpha[q] = A;
    a.T_final[q] = T;
    a.n_contrib[q] = last;
    if (kStats) {
      a.stats[q] = nscan;
      a.stats[HW + q] = ncon;
    }
  }
}

}  // namespace gs

extern "C" int gs_render_fwd(gs_proj pr, const int32_t *sorted_idx, const int32_t *tile_range, gs_camera cam,
                             float *color, float *depth, float *alpha, float *T_final, int32_t *n_contrib,
                             int32_t *stats, void *stream) {
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
            cam.width, cam.height, tiles_x(cam), color, depth, alpha, T_final, n_contrib, stats};
  const int T = tiles_x(cam) * tiles_y(cam);
  if (stats)
    k_render_fwd<true><<<T, kTilePx, 0, as_stream(stream)>>>(a);
  else
    k_render_fwd<false><<<T, kTilePx, 0, as_stream(stream)>>>(a);
  return check_launch("gs_render_fwd");
}
