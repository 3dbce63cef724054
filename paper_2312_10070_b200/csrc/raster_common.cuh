// raster_common.cuh — tile/thread geometry and the alpha evaluation shared by
// gs_render_fwd and gs_render_bwd (H5: both kernels must take bit-identical
// alpha decisions).  Citations as in gs_internal.cuh.
#pragma once

#include "gs_internal.cuh"

namespace gs {

// One CTA per 16x16 tile; every thread owns PX adjacent pixels of one row:
// lane -> columns PX*(lane % (16/PX)) .. +PX-1, row (2 PX) w + lane / (16/PX).
// A warp covers a 16 x (2 PX) strip; a tile has 8/PX warps.  The PX pixels
// share dy, so the row terms of the quadratic form are evaluated once per
// (thread, entry).  The forward uses PX = 2 (short per-warp critical path),
// the backward PX = 4 (half the warp reductions per pixel).
constexpr int kBatch = 128;  // records staged per shared-memory batch

template <int PX>
struct Geo {
  static constexpr int kThreads = kTilePx / PX;
  static constexpr int kWarps = kThreads / 32;
  static constexpr int kLanesPerRow = kTile / PX;
  static constexpr int kRows = 32 / kLanesPerRow;  // rows per warp strip
  static constexpr int kRecPerThread = kBatch / kThreads;
};

struct PixGeom {
  int px0, py;  // first pixel of the thread (absolute)
  float fpx0;   // tile-local column of the first pixel
  float fpy;    // tile-local row
  bool row_in;  // py < H
};

template <int PX>
__device__ __forceinline__ PixGeom pix_geom(int tx, int ty, int H) {
  using G = Geo<PX>;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  PixGeom g;
  const int lx = (lane % G::kLanesPerRow) * PX, ly = w * G::kRows + lane / G::kLanesPerRow;
  g.px0 = tx * kTile + lx;
  g.py = ty * kTile + ly;
  g.fpx0 = float(lx);
  g.fpy = float(ly);
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

// Bit w set iff the box meets warp w's strip [0, 15] x [R w, R w + R - 1].
template <int PX>
__device__ __forceinline__ unsigned box_strip_mask(float4 b) {
  using G = Geo<PX>;
  if (!(b.y >= 0.f && b.x <= float(kTile - 1))) return 0u;
  unsigned m = 0u;
#pragma unroll
  for (int w = 0; w < G::kWarps; ++w) {
    const float y0 = float(w * G::kRows), y1 = y0 + float(G::kRows - 1);
    if (b.w >= y0 && b.z <= y1) m |= 1u << w;
  }
  return m;
}

// This warp's hit bitmaps over a staged batch of kBatch entries: word h has
// bit l set iff entry 32 h + l hits the warp's strip (4 ballots per batch).
__device__ __forceinline__ void warp_hits(const unsigned char *s_mask, int cnt, unsigned hits[kBatch / 32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int h = 0; h < kBatch / 32; ++h) {
    const int j = h * 32 + lane;
    hits[h] = __ballot_sync(0xffffffffu, j < cnt && ((s_mask[j] >> w) & 1u));
  }
}

}  // namespace gs
