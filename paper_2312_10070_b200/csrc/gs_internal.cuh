// gs_internal.cuh — shared device/host helpers of the CUDA path (never used by
// the oracle).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n,
// R# = DESIGN.md §3 readings.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gs.h"

namespace gs {

constexpr int kTile = GS_TILE;
constexpr int kTilePx = kTile * kTile;  // 256 pixels per tile
constexpr float kAlphaMax = GS_ALPHA_MAX;
constexpr float kAlphaMin = GS_ALPHA_MIN;
constexpr float kTEps = GS_T_EPS;
// exponent pre-test: for e < kExpSkip, 2^e < 1/255 by a relative gap of
// 4e-4 >> MUFU.EX2 error (2^-22), so the pre-test never changes a decision.
constexpr float kExpSkip = -7.9950f;
// 0.5 * log2(e): sigma * log2(e) = (a' dx + b' dy)^2 + (d' dy)^2 (H2b)
constexpr double kHalfLog2e = 0.72134752044448170368;

// ---- host-side helpers (abi.cpp) -------------------------------------------
void set_error(const char *fmt, ...);
int check_launch(const char *what);
bool camera_ok(const gs_camera &c);
inline int tiles_x(const gs_camera &c) { return (c.width + kTile - 1) / kTile; }
inline int tiles_y(const gs_camera &c) { return (c.height + kTile - 1) / kTile; }
inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The single alpha evaluation used by BOTH gs_render_fwd and gs_render_bwd
// (H5: bit-identical replay).  Eq. 4: alpha~ = o exp(-sigma),
// sigma = 1/2 Delta^T conic Delta, evaluated as
//   log2 alpha~ = log2 o - (a' dx + b' dy)^2 - (d' dy)^2
// with tile-local fp32 offsets (H2) and explicit round-to-nearest intrinsics
// so no contraction can differ between the two kernels.
// Returns the exponent e; alpha~ = 2^e.
__device__ __forceinline__ float alpha_exponent(float4 coef, float ul, float vl, float fpx,
                                                float fpy, float &dx, float &dy) {
  dx = __fsub_rn(ul, fpx);
  dy = __fsub_rn(vl, fpy);
  float y2 = __fmul_rn(coef.z, dy);
  float y1 = __fmaf_rn(coef.x, dx, __fmul_rn(coef.y, dy));
  float e = __fmaf_rn(-y2, y2, coef.w);
  return __fmaf_rn(-y1, y1, e);
}

// alpha = min(alpha~, 0.999); returns true iff the entry composites
// (alpha >= 1/255, R11).  alpha_t receives alpha~.
__device__ __forceinline__ bool alpha_decide(float e, float &alpha, float &alpha_t) {
  if (e < kExpSkip) return false;
  alpha_t = ex2_approx(e);
  alpha = fminf(alpha_t, kAlphaMax);
  return alpha >= kAlphaMin;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void count_add(int64_t *p, unsigned long long v) {
  if (v) atomicAdd(reinterpret_cast<unsigned long long *>(p), v);
}

}  // namespace gs
