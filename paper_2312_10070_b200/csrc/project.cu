// project.cu — S1 gs_project: EWA projection (Eqs. 1-2).
//
// One thread per Gaussian, coalesced float4 SoA loads.  The decision path
// (p, u, v, Sigma^I, alpha >= 1/255 box, rect, depth key) is evaluated in IEEE
// fp64 in the operation order documented in DESIGN.md §3 R1.  This file is
// compiled with --fmad=false so no multiply-add is contracted: with correctly
// rounded +,-,*,/,sqrt the tile rects and sort keys are reproducible
// bit-for-bit (only exp() may differ by an ulp from another libm).
#include "gs_internal.cuh"

namespace gs {

struct ViewD {
  double R[9], t[3];
};

// camera fields promoted to fp64 once on the host (exact)
struct CamD {
  double fx, fy, cx, cy, zn, zf;
};

#ifndef PROJ_MINB
#define PROJ_MINB 4
#endif
__global__ void __launch_bounds__(256, PROJ_MINB) k_project(gs_params p, const gs_view *__restrict__ view,
                                                 CamD cam, int TX, int TY, gs_proj out,
                                                 gs_counters *cnt) {
  pdl_begin();
  // the view, promoted to fp64 once per block (exact)
  __shared__ ViewD sV;
  if (threadIdx.x < 12) {
    const float f = __ldg(threadIdx.x < 9 ? &view->R[threadIdx.x] : &view->t[threadIdx.x - 9]);
    (threadIdx.x < 9 ? sV.R[threadIdx.x] : sV.t[threadIdx.x - 9]) = (double)f;
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool culled = true, nonfinite = false;
  if (i < p.n) {
    const ViewD &V = sV;
    const float4 mo = __ldg(reinterpret_cast<const float4 *>(p.mean_opa) + i);
    const float4 qf = __ldg(reinterpret_cast<const float4 *>(p.quat) + i);
    const float4 lf = __ldg(reinterpret_cast<const float4 *>(p.logscale) + i);
    const double mu[3] = {mo.x, mo.y, mo.z};
    const double qin[4] = {qf.x, qf.y, qf.z, qf.w};
    // p = R mu + t (Eq. 1's T_wc)
    double pc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
      pc[r] = ((V.R[3 * r] * mu[0] + V.R[3 * r + 1] * mu[1]) + V.R[3 * r + 2] * mu[2]) + V.t[r];
    const double qn = sqrt(((qin[0] * qin[0] + qin[1] * qin[1]) + qin[2] * qin[2]) + qin[3] * qin[3]);
    const double x = pc[0], y = pc[1], z = pc[2];
    const double zn = cam.zn, zf = cam.zf;
    if (!isfinite(x) || !isfinite(y) || !isfinite(z) || !isfinite(qn) || !(qn > 0.0)) {
      nonfinite = true;
    } else if (z >= zn && z <= zf) {  // near/far cull (R5)
      // Sigma = (R_q S)(R_q S)^T
      const double w = qin[0] / qn, qx = qin[1] / qn, qy = qin[2] / qn, qz = qin[3] / qn;
      double Rq[9];
      Rq[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
      Rq[1] = 2.0 * (qx * qy - w * qz);
      Rq[2] = 2.0 * (qx * qz + w * qy);
      Rq[3] = 2.0 * (qx * qy + w * qz);
      Rq[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
      Rq[5] = 2.0 * (qy * qz - w * qx);
      Rq[6] = 2.0 * (qx * qz - w * qy);
      Rq[7] = 2.0 * (qy * qz + w * qx);
      Rq[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
      const double s[3] = {exp((double)lf.x), exp((double)lf.y), exp((double)lf.z)};
      double M[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M[3 * r + c] = Rq[3 * r + c] * s[c];
      double Sig[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          Sig[3 * r + c] = (M[3 * r] * M[3 * c] + M[3 * r + 1] * M[3 * c + 1]) + M[3 * r + 2] * M[3 * c + 2];
      // pinhole pi (R4): u = fx x / z + cx
      const double fx = cam.fx, fy = cam.fy;
      const double u = (fx * x) / z + cam.cx;
      const double v = (fy * y) / z + cam.cy;
      // unclamped EWA Jacobian (Eq. 2, R6)
      const double z2 = z * z;
      const double J0 = fx / z, J2 = -(fx * x) / z2, J4 = fy / z, J5 = -(fy * y) / z2;
      // Sigma_c = R Sigma R^T
      double W[9], Sc[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          W[3 * r + c] = (V.R[3 * r] * Sig[c] + V.R[3 * r + 1] * Sig[3 + c]) + V.R[3 * r + 2] * Sig[6 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          Sc[3 * r + c] = (W[3 * r] * V.R[3 * c] + W[3 * r + 1] * V.R[3 * c + 1]) + W[3 * r + 2] * V.R[3 * c + 2];
      // Sigma^I = J Sigma_c J^T + 0.3 I (R7)
      double T0[3], T1[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        T0[c] = J0 * Sc[c] + J2 * Sc[6 + c];
        T1[c] = J4 * Sc[3 + c] + J5 * Sc[6 + c];
      }
      const double dil = (double)GS_DILATION;
      const double a = (T0[0] * J0 + T0[2] * J2) + dil;
      const double b = T0[1] * J4 + T0[2] * J5;
      const double c = (T1[1] * J4 + T1[2] * J5) + dil;
      const double det = a * c - b * b;
      if (!(det > 0.0) || !isfinite(det) || !isfinite(u) || !isfinite(v)) {
        nonfinite = true;  // singular Sigma^I
      } else {
        // conic (an output, not a decision): one reciprocal
        const double idet = 1.0 / det;
        const double A = c * idet, B = -b * idet, C = a * idet;
        // tile membership (R8'): tiles meeting the box of the region where
        // o exp(-sigma) >= 1/255, sigma <= tau = ln(o / alpha_min): half-widths
        // sqrt(2 tau a), sqrt(2 tau c); no tile when tau <= 0
        const double o = 1.0 / (1.0 + exp(-(double)mo.w));  // sigmoid (R18)
        const double tau = log(o / (double)GS_ALPHA_MIN);
        int x0 = 0, x1 = -1, y0 = 0, y1 = -1;
        if (tau > 0.0) {
          const double hx = sqrt((2.0 * tau) * a), hy = sqrt((2.0 * tau) * c);
          x0 = max((int)floor((u - hx) / kTile), 0);
          x1 = min((int)floor((u + hx) / kTile), TX - 1);
          y0 = max((int)floor((v - hy) / kTile), 0);
          y1 = min((int)floor((v + hy) / kTile), TY - 1);
        }
        if (x0 <= x1 && y0 <= y1) {
          culled = false;
          const float4 cf = __ldg(reinterpret_cast<const float4 *>(p.rgb) + i);
          reinterpret_cast<double2 *>(out.uv)[i] = make_double2(u, v);
          reinterpret_cast<float4 *>(out.conic_o)[i] = make_float4((float)A, (float)B, (float)C, (float)o);
          // H2b Cholesky coefficients, pre-scaled by sqrt(log2(e)/2):
          // a' = sqrt(K A), b' = a' B / A = K B / a', d' = sqrt(K (AC - B^2)/A) = sqrt(K / c)
          // the compositing coefficients (outputs, not decisions; the forward
          // and backward both read these same fp32 values) in fp32 from the
          // fp64 conic: a' = sqrt(K A), b' = K B / a', d' = sqrt(K / c), log2 o
          const float Kf = float(kHalfLog2e);
          const float ap = sqrtf(Kf * float(A));
          reinterpret_cast<float4 *>(out.coef)[i] =
              make_float4(ap, Kf * float(B) / ap, sqrtf(Kf / float(c)), log2f(float(o)));
          reinterpret_cast<float4 *>(out.rgbz)[i] = make_float4(cf.x, cf.y, cf.z, (float)z);
          out.depth[i] = (float)z;  // RN(p_z): the sort key (R10)
          reinterpret_cast<short4 *>(out.rect)[i] = make_short4((short)x0, (short)y0, (short)x1, (short)y1);
          out.tiles_touched[i] = (x1 - x0 + 1) * (y1 - y0 + 1);
        }
      }
    }
    if (culled) {
      out.depth[i] = __int_as_float(0x7f800000);
      reinterpret_cast<short4 *>(out.rect)[i] = make_short4(0, 0, -1, -1);
      out.tiles_touched[i] = 0;
    }
  } else {
    culled = false;
  }
  if (cnt) {
    const unsigned nc = __popc(__ballot_sync(0xffffffffu, culled));
    const unsigned nn = __popc(__ballot_sync(0xffffffffu, nonfinite));
    if ((threadIdx.x & 31) == 0) {
      count_add(&cnt->n_culled, nc);
      count_add(&cnt->n_nonfinite, nn);
    }
  }
}

}  // namespace gs

extern "C" int gs_project(gs_params p, const gs_view *view, gs_camera cam, gs_proj out,
                          gs_counters *cnt, void *stream) {
  using namespace gs;
  if (p.n < 0 || !view || !camera_ok(cam)) {
    set_error("gs_project: invalid argument (n=%d, view=%p, camera ok=%d)", p.n, (const void *)view,
              (int)camera_ok(cam));
    return GS_ERR_INVALID_ARG;
  }
  if (tiles_x(cam) > 32767 || tiles_y(cam) > 32767) {
    set_error("gs_project: image too large for int16 tile rects");
    return GS_ERR_INVALID_ARG;
  }
  if (p.n == 0) return GS_OK;
  const void *ptrs[] = {p.mean_opa, p.quat, p.logscale, p.rgb, out.uv, out.conic_o, out.coef, out.rgbz};
  for (const void *q : ptrs)
    if (!q || !aligned16(q)) {
      set_error("gs_project: null or misaligned (16 B) array");
      return GS_ERR_INVALID_ARG;
    }
  if (!out.depth || !out.rect || !out.tiles_touched || (reinterpret_cast<uintptr_t>(out.rect) & 7u)) {
    set_error("gs_project: null depth/rect/tiles_touched or misaligned rect");
    return GS_ERR_INVALID_ARG;
  }
  const int threads = 256;
  const int blocks = (p.n + threads - 1) / threads;
  const CamD cd{cam.fx, cam.fy, cam.cx, cam.cy, cam.z_near, cam.z_far};
  launch_pdl(k_project, dim3(blocks), dim3(threads), 0, as_stream(stream), p, view, cd, tiles_x(cam), tiles_y(cam),
             out, cnt);
  return check_launch("gs_project");
}
