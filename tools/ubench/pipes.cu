// Pipe-throughput microbenchmark (B200): FFMA vs FFMA2 vs FADD2/FMUL2 vs MUFU.EX2 vs FMNMX.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2u(float2 v){ return *reinterpret_cast<u64*>(&v);}
__device__ __forceinline__ float2 u2f(u64 v){ return *reinterpret_cast<float2*>(&v);}
constexpr int ITERS = 4096;
__global__ void k_ffma(float *out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma_reg(float *out, float a, float b) {  // 3-register form (a, b in regs varying)
  float x[8], av = a + threadIdx.x * 1e-9f, bv = b - threadIdx.x * 1e-9f;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], av, bv);
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float *out, float a, float b) {
  u64 x[8];
  float av = a + threadIdx.x * 1e-9f, bv = b - threadIdx.x * 1e-9f;
  u64 A = f2u(make_float2(av, av)), B = f2u(make_float2(bv, bv));
  for (int i = 0; i < 8; ++i) x[i] = f2u(make_float2(threadIdx.x + i, i));
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 v = u2f(x[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ex2(float *out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -(threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix(float *out, float a, float b) {  // 1 ex2 per 4 ffma
  float x[8], y[8];
  for (int i = 0; i < 8; ++i) { x[i] = -(threadIdx.x + i) * 1e-3f; y[i] = i; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      y[i] = fmaf(y[i], a, b); y[i] = fmaf(y[i], a, b); y[i] = fmaf(y[i], a, b); y[i] = fmaf(y[i], a, b);
    }
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i] + y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fmnmx(float *out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  float av = a + threadIdx.x;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("min.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(av));
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename K>
void run(const char *name, K k, int ops_per_iter_lane, float *d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 8, threads = 256;
  k<<<blocks, threads>>>(d, 0.999f, 1e-3f);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(d, 0.999f, 1e-3f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = double(blocks) * threads * ITERS * 8 * ops_per_iter_lane;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-10s %8.3f ms  %8.1f Gop/s  %6.1f lane-ops/clk/SM (at %d MHz nominal)\n", name, ms, ops / ms / 1e6,
         ops / cyc / 148, clk / 1000);
}
int main() {
  float *d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  run("ffma_imm", k_ffma, 1, d);
  run("ffma_reg", k_ffma_reg, 1, d);
  run("ffma2", k_ffma2, 2, d);
  run("ex2", k_ex2, 1, d);
  run("ex2+4ffma", k_mix, 5, d);
  run("fmnmx", k_fmnmx, 1, d);
  return 0;
}
