// rgbd.cu — gs_unpack_rgbd: an RGB-D frame in the format of the paper's
// sensors and datasets ("the RGBD frame", "the input color and
// depth map at frame i", "trajectories from an RGBD sensor"): 8-bit
// RGB, interleaved [H][W][3], and 16-bit depth [H][W] in units of
// depth_scale metres, into the fp32 planar targets of gs_loss / the
// tracking loss:  color[c][q] = rgb[q][c] / 255,  depth[q] = d[q] * scale.
// HBM-bound (5 B read + 16 B written per pixel); 4 pixels per thread with
// vector loads and stores when the sizes and pointers allow it.
#include <algorithm>

#include "gs_internal.cuh"

namespace gs {

constexpr int kUnpackThreads = 256;

template <bool kVec>
__global__ void __launch_bounds__(kUnpackThreads) k_unpack_rgbd(const uint8_t *__restrict__ rgb,
                                                                const uint16_t *__restrict__ d16, int64_t HW,
                                                                float scale, float *__restrict__ color,
                                                                float *__restrict__ depth, unsigned *valid) {
  unsigned nv = 0;  // valid depths (D* > 0 <=> d16 > 0) of this thread, for gs_loss_scales' |V|
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; 4 * t < HW; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q0 = 4 * t;
    if (kVec) {
      const uint32_t *c4 = reinterpret_cast<const uint32_t *>(rgb) + 3 * t;  // 12 bytes: pixels q0..q0+3
      const uint2 dd = __ldg(reinterpret_cast<const uint2 *>(d16) + t);
      const uint32_t w[3] = {__ldg(c4), __ldg(c4 + 1), __ldg(c4 + 2)};
      float v[12];
#pragma unroll
      for (int b = 0; b < 12; ++b)  // byte b = 3 * pixel + channel; IEEE division, as the oracle
        v[b] = __fdiv_rn(float((w[b >> 2] >> (8 * (b & 3))) & 0xffu), 255.f);
#pragma unroll
      for (int ch = 0; ch < 3; ++ch)
        reinterpret_cast<float4 *>(color + ch * HW)[t] = make_float4(v[ch], v[3 + ch], v[6 + ch], v[9 + ch]);
      reinterpret_cast<float4 *>(depth)[t] =
          make_float4(__fmul_rn(float(dd.x & 0xffffu), scale), __fmul_rn(float(dd.x >> 16), scale),
                      __fmul_rn(float(dd.y & 0xffffu), scale), __fmul_rn(float(dd.y >> 16), scale));
      nv += ((dd.x & 0xffffu) != 0u) + ((dd.x >> 16) != 0u) + ((dd.y & 0xffffu) != 0u) + ((dd.y >> 16) != 0u);
    } else {
      for (int64_t q = q0; q < q0 + 4 && q < HW; ++q) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) color[ch * HW + q] = __fdiv_rn(float(rgb[3 * q + ch]), 255.f);
        depth[q] = __fmul_rn(float(d16[q]), scale);
        nv += d16[q] != 0;
      }
    }
  }
  if (valid) {  // one atomic per block (integer counts: the total is order-independent)
    __shared__ unsigned sw[kUnpackThreads / 32];
    nv = __reduce_add_sync(0xffffffffu, nv);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = nv;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned b = 0;
      for (int k = 0; k < kUnpackThreads / 32; ++k) b += sw[k];
      if (b) atomicAdd(valid, b);
    }
  }
}

// gs_loss_scales' values from the valid-depth count (same formulas)
__global__ void k_unpack_scales(float *scales, int64_t HW, float lc, float ld) {
  unsigned *cnt = reinterpret_cast<unsigned *>(scales + 3);
  const unsigned nv = *cnt;
  scales[0] = float(double(lc) / (3.0 * double(HW)));
  scales[1] = nv ? float(double(ld) / double(nv)) : 0.f;
  scales[2] = float(nv);
  scales[3] = 0.f;
}

}  // namespace gs

extern "C" int gs_unpack_rgbd(gs_camera cam, const uint8_t *rgb, const uint16_t *depth16, float depth_scale,
                              float *tgt_color, float *tgt_depth, float *scales, float lambda_color,
                              float lambda_depth, void *stream) {
  using namespace gs;
  if (!camera_ok(cam) || !rgb || !depth16 || !tgt_color || !tgt_depth || !(depth_scale > 0.f) ||
      (scales && !(lambda_color >= 0.f && lambda_depth >= 0.f))) {
    set_error("gs_unpack_rgbd: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  const int64_t HW = int64_t(cam.width) * cam.height;
  const bool vec = HW % 4 == 0 && (reinterpret_cast<uintptr_t>(rgb) & 3u) == 0 &&
                   (reinterpret_cast<uintptr_t>(depth16) & 7u) == 0 && aligned16(tgt_color) && aligned16(tgt_depth);
  const int64_t quads = (HW + 3) / 4;
  const int blocks = int(std::min<int64_t>((quads + kUnpackThreads - 1) / kUnpackThreads, 148 * 16));
  cudaStream_t s = as_stream(stream);
  unsigned *valid = scales ? reinterpret_cast<unsigned *>(scales + 3) : nullptr;  // the count, in scales[3]
  if (valid) cudaMemsetAsync(valid, 0, sizeof(unsigned), s);
  if (vec)
    k_unpack_rgbd<true><<<blocks, kUnpackThreads, 0, s>>>(rgb, depth16, HW, depth_scale, tgt_color, tgt_depth, valid);
  else
    k_unpack_rgbd<false><<<blocks, kUnpackThreads, 0, s>>>(rgb, depth16, HW, depth_scale, tgt_color, tgt_depth, valid);
  if (scales) k_unpack_scales<<<1, 1, 0, s>>>(scales, HW, lambda_color, lambda_depth);
  return check_launch("gs_unpack_rgbd");
}
