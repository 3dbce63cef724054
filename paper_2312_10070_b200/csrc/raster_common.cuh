// raster_common.cuh — tile/thread geometry and the alpha evaluation shared by
// gs_render_fwd and gs_render_bwd (H5: both kernels must take bit-identical
// alpha decisions).  Citations as in gs_internal.cuh.
#pragma once

#include "gs_internal.cuh"

namespace gs {

// One CTA per 16x16 tile; every thread owns PX adjacent pixels of one row.
// A warp covers a WX x (32 PX / WX) block of the tile (WX = 8 or 16); warps
// tile the 16x16 tile row-major.  The PX pixels of a thread share dy, so the
// row terms of the quadratic form are evaluated once per (thread, entry), and
// they are processed in pairs with the packed fp32x2 pipe (FFMA2).
//   forward  : PX = 2, WX = 8  -> 4 warps, 8x8 blocks
//   backward : PX = 4, WX = 16 -> 2 warps, 16x8 strips
constexpr int kBatch = 128;  // records staged per shared-memory batch

template <int PX, int WX>
struct Geo {
  static_assert(PX % 2 == 0, "pixels are processed in pairs");
  static constexpr int kThreads = kTilePx / PX;
  static constexpr int kWarps = kThreads / 32;
  static constexpr int kLanesPerRow = WX / PX;
  static constexpr int kRows = 32 / kLanesPerRow;  // rows per warp block
  static constexpr int kAcross = kTile / WX;       // warp blocks per tile row
  static constexpr int kRecPerThread = kBatch / kThreads;
  static_assert(kWarps * WX * kRows == kTilePx, "warp blocks must tile the tile");
  // tile-local origin of warp w's block
  static __host__ __device__ constexpr int bx(int w) { return (w % kAcross) * WX; }
  static __host__ __device__ constexpr int by(int w) { return (w / kAcross) * kRows; }
};

struct PixGeom {
  int px0, py;  // first pixel of the thread (absolute)
  float fpx0;   // tile-local column of the first pixel
  float fpy;    // tile-local row
  bool row_in;  // py < H
};

// w: the warp block of the tile this warp owns (default: its warp index)
template <class G>
__device__ __forceinline__ PixGeom pix_geom(int tx, int ty, int H, int w = int(threadIdx.x >> 5)) {
  const int lane = threadIdx.x & 31;
  PixGeom g;
  const int lx = G::bx(w) + (lane % G::kLanesPerRow) * (kTilePx / G::kThreads);
  const int ly = G::by(w) + lane / G::kLanesPerRow;
  g.px0 = tx * kTile + lx;
  g.py = ty * kTile + ly;
  g.fpx0 = float(lx);
  g.fpy = float(ly);
  g.row_in = g.py < H;
  return g;
}

// log2 alpha~ = log2 o - y1^2 - y2^2 with y1 = a' (u_l - x) + b' (v_l - y),
// y2 = d' (v_l - y): the H2b Cholesky form of sigma, in tile-local fp32
// offsets (H2).  Staged once per entry (EntryTerms):
//   p = (a', b', d', K = a' u_l + b' v_l),  q = (DV = d' v_l, log2 o)
// per (thread, entry) row terms (3 FFMA):
//   c0 = K - b' y,  y2 = DV - d' y,  e0 = log2 o - y2^2
// and per pixel x (2 FFMA, as FFMA2 over a pixel pair):
//   y1 = c0 - a' x,  e = e0 - y1^2.
// Explicit round-to-nearest intrinsics and FMA-only chains: no contraction
// can differ between the forward and the backward kernel (an FFMA2 lane is
// the correctly rounded FMA, identical to the scalar one).
struct EntryTerms {
  float4 p;
  float2 q;
};

__device__ __forceinline__ EntryTerms entry_terms(float4 coef, float ul, float vl) {
  EntryTerms t;
  t.p = make_float4(coef.x, coef.y, coef.z, __fmaf_rn(coef.x, ul, __fmul_rn(coef.y, vl)));
  t.q = make_float2(__fmul_rn(coef.z, vl), coef.w);
  return t;
}

struct RowTerms {
  float2 na, c0, e0;  // broadcast pairs: -a', c0, e0
};

__device__ __forceinline__ RowTerms row_terms(float4 p, float2 q, float fpy) {
  const float c0 = __fmaf_rn(-p.y, fpy, p.w);
  const float y2 = __fmaf_rn(-p.z, fpy, q.x);
  const float e0 = __fmaf_rn(-y2, y2, q.y);
  RowTerms r;
  r.na = make_float2(-p.x, -p.x);
  r.c0 = make_float2(c0, c0);
  r.e0 = make_float2(e0, e0);
  return r;
}

// exponent at the pixel pair x = (fx.x, fx.y)
__device__ __forceinline__ float2 pair_exponent(const RowTerms &r, float2 fx) {
  const float2 y1 = __ffma2_rn(r.na, fx, r.c0);
  return __ffma2_rn(make_float2(-y1.x, -y1.y), y1, r.e0);
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

// Bit w set iff the box meets warp w's block.
template <class G>
__device__ __forceinline__ unsigned box_block_mask(float4 b) {
  unsigned m = 0u;
#pragma unroll
  for (int w = 0; w < G::kWarps; ++w) {
    const float x0 = float(G::bx(w)), y0 = float(G::by(w));
    if (b.y >= x0 && b.x <= x0 + float(16 / G::kAcross - 1) && b.w >= y0 && b.z <= y0 + float(G::kRows - 1))
      m |= 1u << w;
  }
  return m;
}

// Exact culling of an entry against the warp blocks (a refinement of the box
// test): the minimum over the continuous block rectangle [x0, x1] x [y0, y1]
// (tile-local pixel centres) of E = y1^2 + y2^2 = (a' dx + b' dy)^2 +
// (d' dy)^2, dx = u_l - x, dy = v_l - y, compared with R^2 = log2 o -
// kExpSkip.  The rectangle contains every pixel centre of the block, so a
// block with min E > R^2 has e = log2 o - E < kExpSkip < kExpMin at all of its
// pixels (the kExpSkip margin, 6.5e-4, covers the fp32 rounding of E there
// and here): dropping it never changes a decision.  The minimum of the convex
// E is 0 if (dx, dy) = 0 lies in the rectangle, else on an edge: on dy = Y at
// dx = -b' Y / a', on dx = X at dy = -a' b' X / (b'^2 + d'^2), clamped.
__device__ __forceinline__ float rect_min_E(float a, float b, float d, float ia, float ibd, float dx0, float dx1,
                                            float dy0, float dy1) {
  if (dx0 <= 0.f && dx1 >= 0.f && dy0 <= 0.f && dy1 >= 0.f) return 0.f;
  const float d2 = d * d;
  auto edge_y = [&](float y) {
    const float x = fminf(fmaxf(-b * y * ia, dx0), dx1);
    const float u = fmaf(a, x, b * y);
    return fmaf(u, u, d2 * y * y);
  };
  auto edge_x = [&](float x) {
    const float y = fminf(fmaxf(-a * b * x * ibd, dy0), dy1);
    const float u = fmaf(a, x, b * y);
    return fmaf(u, u, d2 * y * y);
  };
  return fminf(fminf(edge_y(dy0), edge_y(dy1)), fminf(edge_x(dx0), edge_x(dx1)));
}

// Bit w set iff the entry can pass the exponent pre-test at some pixel of
// warp block w: the box test, then the exact rectangle test.
template <class G>
__device__ __forceinline__ unsigned entry_block_mask(float4 coef, float ul, float vl) {
  const float R2 = coef.w - kExpSkip;
  const unsigned m = box_block_mask<G>(entry_box(coef, ul, vl));
  if (!m) return 0u;
  const float ia = 1.0f / coef.x, ibd = 1.0f / fmaf(coef.y, coef.y, coef.z * coef.z);
  unsigned r = 0u;
#pragma unroll
  for (int w = 0; w < G::kWarps; ++w) {
    if (!((m >> w) & 1u)) continue;
    const float x0 = float(G::bx(w)), y0 = float(G::by(w));
    const float x1 = x0 + float(16 / G::kAcross - 1), y1 = y0 + float(G::kRows - 1);
    if (rect_min_E(coef.x, coef.y, coef.z, ia, ibd, ul - x1, ul - x0, vl - y1, vl - y0) <= R2) r |= 1u << w;
  }
  return r;
}

// This warp's hit list over a staged batch of B entries: the indices
// (ascending) of the entries j < cnt whose mask has bit w (default: the warp
// index), written to list[0..n), followed by `sentinel` at list[n].  Returns n.
template <int B = kBatch, class L>
__device__ __forceinline__ int warp_hit_list(const unsigned char *s_mask, int cnt, L *list, int sentinel,
                                             int w = int(threadIdx.x >> 5)) {
  const int lane = threadIdx.x & 31;
  int n = 0;
#pragma unroll
  for (int h = 0; h < B / 32; ++h) {
    const int j = h * 32 + lane;
    const bool hit = j < cnt && ((s_mask[j] >> w) & 1u);
    const unsigned b = __ballot_sync(0xffffffffu, hit);
    if (hit) list[n + __popc(b & lanemask_lt())] = (L)j;
    n += __popc(b);
  }
  if (lane == 0) list[n] = (L)sentinel;
  __syncwarp();
  return n;
}

}  // namespace gs
