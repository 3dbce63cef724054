// raster_common.cuh — tile/thread geometry and the alpha evaluation shared by
// gs_render_fwd and gs_render_bwd (H5: both kernels must take bit-identical
// alpha decisions).  Citations as in gs_internal.cuh.
#pragma once

#include "gs_internal.cuh"

namespace gs {

// One CTA per 16x16 tile, 4 warps; every thread owns 2 adjacent pixels of one
// row: lane -> columns 2*(lane&7), +1, row 4*warp + (lane>>3).  A warp covers a
// 16x4 strip.  The 2 pixels share dy, so the row terms of the quadratic form
// are evaluated once per (thread, entry).
constexpr int kRThreadsTile = 128;
constexpr int kPxPerThread = 2;
constexpr int kWarpRows = 4;
constexpr int kBatch = 128;  // records staged per shared-memory batch (1 per thread)

struct PixGeom {
  int px0, py;  // first pixel of the thread (absolute)
  float fpx0;   // tile-local column of the first pixel
  float fpy;    // tile-local row
  float wy0;    // first tile-local row of the warp's strip
  bool row_in;  // py < H
};

__device__ __forceinline__ PixGeom pix_geom(int tx, int ty, int H) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  PixGeom g;
  const int lx = (lane & 7) * kPxPerThread, ly = w * kWarpRows + (lane >> 3);
  g.px0 = tx * kTile + lx;
  g.py = ty * kTile + ly;
  g.fpx0 = float(lx);
  g.fpy = float(ly);
  g.wy0 = float(w * kWarpRows);
  g.row_in = g.py < H;
  return g;
}

// Per-(thread, entry) row terms of log2 alpha~ = log2 o - y1^2 - y2^2 with
// y1 = a' (u_l - x) + b' (v_l - y), y2 = d' (v_l - y), tile-local fp32
// offsets (H2) and the H2b coefficients (a', b', d', log2 o):
//   e0 = log2 o - y2^2,  c0 = a' u_l + b' (v_l - y)
// and per pixel x:  y1 = c0 - a' x,  e = e0 - y1^2.
// Explicit round-to-nearest intrinsics: no contraction can differ between the
// forward and the backward kernel.
struct RowTerms {
  float e0, c0, na;  // na = -a'
};

__device__ __forceinline__ RowTerms row_terms(float4 coef, float ul, float vl, float fpy) {
  const float dy = __fsub_rn(vl, fpy);
  const float y2 = __fmul_rn(coef.z, dy);
  RowTerms r;
  r.e0 = __fmaf_rn(-y2, y2, coef.w);
  r.c0 = __fmaf_rn(coef.x, ul, __fmul_rn(coef.y, dy));
  r.na = -coef.x;
  return r;
}

__device__ __forceinline__ float pixel_exponent(const RowTerms &r, float fpx) {
  const float y1 = __fmaf_rn(r.na, fpx, r.c0);
  return __fmaf_rn(-y1, y1, r.e0);
}

// Conservative tile-local box of the region where an entry can pass the
// exponent pre-test e >= kExpSkip, i.e. y1^2 + y2^2 <= R^2 = log2 o - kExpSkip:
// half-widths R sqrt(d'^2 + b'^2) / (a' d') in x and R / d' in y, padded by
// 0.05 px.  Used only to skip work a warp would reject pixel by pixel anyway:
// it never changes a decision.  Empty (x0 > x1) when log2 o < kExpSkip.
__device__ __forceinline__ float4 entry_box(float4 coef, float ul, float vl) {
  const float R2 = coef.w - kExpSkip;
  if (!(R2 > 0.f)) return make_float4(1.f, -1.f, 1.f, -1.f);
  const float R = sqrtf(R2);
  const float hy = R / coef.z + 0.05f;
  const float hx = R * sqrtf(coef.z * coef.z + coef.y * coef.y) / (coef.x * coef.z) + 0.05f;
  return make_float4(ul - hx, ul + hx, vl - hy, vl + hy);
}

// Does the box meet the warp's strip [0, 15] x [wy0, wy0 + kWarpRows - 1]?
__device__ __forceinline__ bool box_hits_strip(float4 b, float wy0) {
  return b.y >= 0.f && b.x <= float(kTile - 1) && b.w >= wy0 && b.z <= wy0 + float(kWarpRows - 1);
}

}  // namespace gs
