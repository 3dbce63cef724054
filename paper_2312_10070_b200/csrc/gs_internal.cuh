// gs_internal.cuh — shared device/host helpers of the CUDA path (never used by
// the oracle).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n,
// R# = DESIGN.md §3 readings.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gs.h"

// Device-side bounds checks of the debug build (libgs_debug.so, compiled with
// -DGS_DEBUG by _build.py): a failed check prints its location and traps (the
// launch fails with a CUDA error).  compute-sanitizer is closed on this pool;
// these checks on every index that a kernel derives from another kernel's
// output are the substitute (tests run under the debug build: profiles/r02).
#ifdef GS_DEBUG
#include <cstdio>
#define GS_ASSERT(c)                                                        \
  do {                                                                      \
    if (!(c)) {                                                             \
      printf("GS_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      __trap();                                                             \
    }                                                                       \
  } while (0)
#else
#define GS_ASSERT(c) ((void)0)
#endif

namespace gs {

constexpr int kTile = GS_TILE;
constexpr int kTilePx = kTile * kTile;  // 256 pixels per tile
constexpr float kAlphaMax = GS_ALPHA_MAX;
constexpr float kAlphaMin = GS_ALPHA_MIN;
constexpr float kTEps = GS_T_EPS;
// The alpha decisions of R11 are taken on the fp32 exponent e (log2 alpha~,
// raster_common.cuh), in both render kernels (R2'):
//   alpha~ >= 1/255 (GS_ALPHA_MIN)  <=>  e >= kExpMin
//   alpha~ >= 0.999 (GS_ALPHA_MAX)  <=>  e >= kExpClamp
// each constant the smallest float >= log2 of the (fp32) threshold, so the
// test is the exact decision for 2^e; no MUFU.EX2 rounding enters it.
constexpr float kExpMin = -7.994353294373e+00f;    // 0xc0ffd1be, log2(1/255f) = -7.99435335...
constexpr float kExpClamp = -1.443398185074e-03f;  // 0xbabd3068, log2(0.999f) = -0.00144339827...
// conservative bound for the entry boxes (below kExpMin by 6.5e-4)
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

// ---- programmatic dependent launch (PDL) ------------------------------------
// The kernels of the path start with pdl_begin(): wait until the preceding
// kernel's grid has completed and its memory is visible (a no-op when the
// kernel was launched without the attribute), then allow the next kernel's
// CTAs to be scheduled.  launch_pdl() launches with the attribute, so a
// kernel's launch and CTA set-up overlap its predecessor's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
  pdl_wait();
  pdl_trigger();
}

#ifndef GS_PDL
#define GS_PDL 1
#endif
template <typename... KArgs, typename... Args>
inline void launch_pdl_if(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                          Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl && GS_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = GS_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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
