// render_bwd.cu — S5 + S6 gs_render_bwd (Eqs. 7-8).
//
// S5 (k_bwd_pixels): one CTA per tile, one pixel per thread.  Every pixel
// replays its composited entries back to front starting from T_final and
// n_contrib, recomputing alpha with the very same alpha_exponent /
// alpha_decide as gs_render_fwd (H5), reconstructing T_j = T_{j+1}/(1-alpha_j)
// and carrying the suffix accumulators of Eq. 8
//   S_X <- alpha_j X_j + (1 - alpha_j) S_X,  dX/dalpha_j = T_j (X_j - S_X)
// for X = colour (3), camera depth, alpha.  Per-entry 2-D gradients are summed
// across the warp with shuffles (skipped when no lane composited the entry)
// and added to the grad2d scratch with one vector red per float4.
//
// S6 (k_bwd_gauss): one thread per visible Gaussian chains the 2-D gradients
// to mean, quaternion, log-scales, opacity logit and colour ("derived as in
// [kerbl]"), and for tracking reduces the pose partials block-wise.
#include "gs_internal.cuh"

namespace gs {

// grad2d record [n][12]: (u, v, A, B), (C, p_z, logit, 0), (r, g, b, 0)
constexpr int kG2 = 12;

__device__ __forceinline__ void red_add_v4(float *addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

struct BwdArgs {
  const double2 *uv;
  const float4 *coef;
  const float4 *rgbz;
  const float4 *conic_o;
  const int32_t *sorted_idx;
  const int2 *tile_range;
  const float *T_final;
  const int32_t *n_contrib;
  const float *dL_dcolor, *dL_ddepth, *dL_dalpha;
  int W, H, TX;
  float *grad2d;
};

template <bool kParams>
__global__ void __launch_bounds__(kTilePx) k_bwd_pixels(BwdArgs a) {
  __shared__ int s_idx[kTilePx];
  __shared__ float2 s_uv[kTilePx];
  __shared__ float4 s_coef[kTilePx];
  __shared__ float4 s_rgbz[kTilePx];
  __shared__ float4 s_conic[kTilePx];
  __shared__ int s_lmax;
  const int tile = blockIdx.x;
  const int tx = tile % a.TX, ty = tile / a.TX;
  const int lx = threadIdx.x & (kTile - 1), ly = threadIdx.x / kTile;
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < a.W && py < a.H;
  const double ox = double(tx * kTile), oy = double(ty * kTile);
  const float fpx = float(lx), fpy = float(ly);
  const int2 range = a.tile_range[tile];
  const size_t HW = size_t(a.W) * a.H, q = size_t(py) * a.W + px;
  float T = 1.f, G0 = 0.f, G1 = 0.f, G2 = 0.f, GD = 0.f, GA = 0.f;
  int last = 0;
  if (inside) {
    T = a.T_final[q];
    last = a.n_contrib[q];
    G0 = a.dL_dcolor[q];
    G1 = a.dL_dcolor[HW + q];
    G2 = a.dL_dcolor[2 * HW + q];
    GD = a.dL_ddepth[q];
    GA = a.dL_dalpha ? a.dL_dalpha[q] : 0.f;
  }
  if (threadIdx.x == 0) s_lmax = 0;
  __syncthreads();
  if (last > 0) atomicMax(&s_lmax, last);
  __syncthreads();
  const int lmax = s_lmax;
  float S0 = 0.f, S1 = 0.f, S2 = 0.f, SD = 0.f, SA = 0.f;  // suffix accumulators (Eq. 8)
  const int lane = threadIdx.x & 31;
  for (int end = lmax; end > 0; end -= kTilePx) {
    const int beg = max(end - kTilePx, 0);
    __syncthreads();
    const int k = beg + threadIdx.x;
    if (k < end) {
      const int g = __ldg(a.sorted_idx + range.x + k);
      const double2 u = __ldg(a.uv + g);
      s_idx[threadIdx.x] = g;
      s_uv[threadIdx.x] = make_float2(float(u.x - ox), float(u.y - oy));
      s_coef[threadIdx.x] = __ldg(a.coef + g);
      s_rgbz[threadIdx.x] = __ldg(a.rgbz + g);
      s_conic[threadIdx.x] = __ldg(a.conic_o + g);
    }
    __syncthreads();
    for (int j = end - beg - 1; j >= 0; --j) {
      const int pos = beg + j;
      float gu = 0.f, gv = 0.f, gA = 0.f, gB = 0.f, gC = 0.f, gz = 0.f, gl = 0.f, gr = 0.f, gg = 0.f, gb = 0.f;
      bool con = false;
      if (pos < last) {
        const float2 ul = s_uv[j];
        float dx, dy, al, at;
        const float e = alpha_exponent(s_coef[j], ul.x, ul.y, fpx, fpy, dx, dy);
        con = alpha_decide(e, al, at);
        if (con) {
          const float4 c = s_rgbz[j];
          const float om = __fsub_rn(1.f, al);
          T = __fdiv_rn(T, om);  // T_j (R16)
          const float w = al * T;
          // dX/dalpha_j = T_j (X_j - S_X) (Eq. 8), chained with dL/dX (Eq. 7)
          const float galpha = T * (G0 * (c.x - S0) + G1 * (c.y - S1) + G2 * (c.z - S2) + GD * (c.w - SD) +
                                    GA * (1.f - SA));
          gz = w * GD;  // dD/dz_j = alpha_j T_j
          if (kParams) {
            gr = w * G0;  // dC/dc_j = alpha_j T_j
            gg = w * G1;
            gb = w * G2;
          }
          S0 = fmaf(al, c.x - S0, S0);
          S1 = fmaf(al, c.y - S1, S1);
          S2 = fmaf(al, c.z - S2, S2);
          SD = fmaf(al, c.w - SD, SD);
          SA = fmaf(al, 1.f - SA, SA);
          if (at < kAlphaMax) {  // a clamped alpha has no gradient (R17)
            const float4 cn = s_conic[j];
            if (kParams) gl = galpha * al * (1.f - cn.w);  // d alpha / d logit = alpha (1 - o)
            const float gs = -al * galpha;                   // d alpha / d sigma = -alpha
            gu = gs * (cn.x * dx + cn.y * dy);
            gv = gs * (cn.y * dx + cn.z * dy);
            gA = 0.5f * gs * dx * dx;
            gB = gs * dx * dy;
            gC = 0.5f * gs * dy * dy;
          }
        }
      }
      if (__ballot_sync(0xffffffffu, con) == 0) continue;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gu += __shfl_down_sync(0xffffffffu, gu, o);
        gv += __shfl_down_sync(0xffffffffu, gv, o);
        gA += __shfl_down_sync(0xffffffffu, gA, o);
        gB += __shfl_down_sync(0xffffffffu, gB, o);
        gC += __shfl_down_sync(0xffffffffu, gC, o);
        gz += __shfl_down_sync(0xffffffffu, gz, o);
        if (kParams) {
          gl += __shfl_down_sync(0xffffffffu, gl, o);
          gr += __shfl_down_sync(0xffffffffu, gr, o);
          gg += __shfl_down_sync(0xffffffffu, gg, o);
          gb += __shfl_down_sync(0xffffffffu, gb, o);
        }
      }
      if (lane == 0) {
        float *dst = a.grad2d + size_t(s_idx[j]) * kG2;
        red_add_v4(dst, gu, gv, gA, gB);
        red_add_v4(dst + 4, gC, gz, gl, 0.f);
        if (kParams) red_add_v4(dst + 8, gr, gg, gb, 0.f);
      }
    }
  }
}

struct GaussArgs {
  gs_params p;
  const gs_view *view;
  float fx, fy;
  const float4 *conic_o;
  const int32_t *tiles_touched;
  float *grad2d;
  float4 *g_mean_opa, *g_quat, *g_logscale, *g_rgb;
  float *pose_partials;
};

template <bool kParams, bool kPose>
__global__ void __launch_bounds__(256) k_bwd_gauss(GaussArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float pose[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) pose[k] = 0.f;
  if (i < a.p.n && __ldg(a.tiles_touched + i) > 0) {
    float R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = __ldg(&a.view->R[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = __ldg(&a.view->t[k]);
    const float4 mo = __ldg(reinterpret_cast<const float4 *>(a.p.mean_opa) + i);
    const float4 qf = __ldg(reinterpret_cast<const float4 *>(a.p.quat) + i);
    const float4 lf = __ldg(reinterpret_cast<const float4 *>(a.p.logscale) + i);
    const float4 cn = __ldg(a.conic_o + i);
    float4 *g2 = reinterpret_cast<float4 *>(a.grad2d) + 3 * i;
    const float4 ga = g2[0], gb = g2[1], gc = g2[2];
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    g2[0] = z4;  // leave the scratch zeroed for the next call
    g2[1] = z4;
    g2[2] = z4;
    const float gu = ga.x, gv = ga.y, gA = ga.z, gB = ga.w, gC = gb.x, gz = gb.y;
    const float mu[3] = {mo.x, mo.y, mo.z};
    float p[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) p[r] = R[3 * r] * mu[0] + R[3 * r + 1] * mu[1] + R[3 * r + 2] * mu[2] + t[r];
    const float x = p[0], y = p[1], z = p[2];
    // Sigma = M M^T, M = R_q S
    const float qn = sqrtf(qf.x * qf.x + qf.y * qf.y + qf.z * qf.z + qf.w * qf.w);
    const float iq = 1.f / qn;
    const float qw = qf.x * iq, qx = qf.y * iq, qy = qf.z * iq, qz = qf.w * iq;
    float Rq[9];
    Rq[0] = 1.f - 2.f * (qy * qy + qz * qz);
    Rq[1] = 2.f * (qx * qy - qw * qz);
    Rq[2] = 2.f * (qx * qz + qw * qy);
    Rq[3] = 2.f * (qx * qy + qw * qz);
    Rq[4] = 1.f - 2.f * (qx * qx + qz * qz);
    Rq[5] = 2.f * (qy * qz - qw * qx);
    Rq[6] = 2.f * (qx * qz - qw * qy);
    Rq[7] = 2.f * (qy * qz + qw * qx);
    Rq[8] = 1.f - 2.f * (qx * qx + qy * qy);
    const float s[3] = {expf(lf.x), expf(lf.y), expf(lf.z)};
    float M[9], Sig[9], W[9], Sc[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) M[3 * r + c] = Rq[3 * r + c] * s[c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) Sig[3 * r + c] = M[3 * r] * M[3 * c] + M[3 * r + 1] * M[3 * c + 1] + M[3 * r + 2] * M[3 * c + 2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) W[3 * r + c] = R[3 * r] * Sig[c] + R[3 * r + 1] * Sig[3 + c] + R[3 * r + 2] * Sig[6 + c];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) Sc[3 * r + c] = W[3 * r] * R[3 * c] + W[3 * r + 1] * R[3 * c + 1] + W[3 * r + 2] * R[3 * c + 2];
    const float iz = 1.f / z, iz2 = iz * iz, iz3 = iz2 * iz;
    const float J0 = a.fx * iz, J2 = -a.fx * x * iz2, J4 = a.fy * iz, J5 = -a.fy * y * iz2;
    // conic -> Sigma^I: G_S2 = -Conic G_M Conic, G_M = [[gA, gB/2], [gB/2, gC]]
    const float A = cn.x, B = cn.y, C = cn.z;
    const float hB = 0.5f * gB;
    const float t00 = A * gA + B * hB, t01 = A * hB + B * gC, t10 = B * gA + C * hB, t11 = B * hB + C * gC;
    const float S00 = -(t00 * A + t01 * B), S01 = -(t00 * B + t01 * C), S11 = -(t10 * B + t11 * C);
    // Sigma^I = J Sigma_c J^T: G_Sc = J^T G_S2 J, G_J = 2 G_S2 J Sigma_c
    // J = [[J0, 0, J2], [0, J4, J5]]
    const float Jm[6] = {J0, 0.f, J2, 0.f, J4, J5};
    const float GS2[4] = {S00, S01, S01, S11};
    float GSc[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float acc = 0.f;
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 2; ++v) acc += Jm[3 * u + r] * GS2[2 * u + v] * Jm[3 * v + c];
        GSc[3 * r + c] = acc;
      }
    float GJ0[6], GJ[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) GJ0[3 * r + c] = GS2[2 * r] * Jm[c] + GS2[2 * r + 1] * Jm[3 + c];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        GJ[3 * r + c] = 2.f * (GJ0[3 * r] * Sc[c] + GJ0[3 * r + 1] * Sc[3 + c] + GJ0[3 * r + 2] * Sc[6 + c]);
    // camera-frame mean p: through (u, v) (Eq. 1), J(p) and the depth term (Eq. 6)
    float gp[3];
    gp[0] = gu * a.fx * iz - GJ[2] * a.fx * iz2;
    gp[1] = gv * a.fy * iz - GJ[5] * a.fy * iz2;
    gp[2] = -gu * a.fx * x * iz2 - gv * a.fy * y * iz2 + gz - GJ[0] * a.fx * iz2 + GJ[2] * 2.f * a.fx * x * iz3 -
            GJ[4] * a.fy * iz2 + GJ[5] * 2.f * a.fy * y * iz3;
    if (kParams) {
      float gmu[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) gmu[c] = R[c] * gp[0] + R[3 + c] * gp[1] + R[6 + c] * gp[2];
      // G_Sigma = R^T G_Sc R; G_M = 2 G_Sigma M
      float tmp[9], GSig[9], GM3[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) tmp[3 * r + c] = R[r] * GSc[c] + R[3 + r] * GSc[3 + c] + R[6 + r] * GSc[6 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) GSig[3 * r + c] = tmp[3 * r] * R[c] + tmp[3 * r + 1] * R[3 + c] + tmp[3 * r + 2] * R[6 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          GM3[3 * r + c] = 2.f * (GSig[3 * r] * M[c] + GSig[3 * r + 1] * M[3 + c] + GSig[3 * r + 2] * M[6 + c]);
      float gls[3], GRq[9];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        gls[k] = s[k] * (GM3[k] * Rq[k] + GM3[3 + k] * Rq[3 + k] + GM3[6 + k] * Rq[6 + k]);
#pragma unroll
        for (int r = 0; r < 3; ++r) GRq[3 * r + k] = GM3[3 * r + k] * s[k];
      }
      // dR(q^)/dq^ contracted with G_Rq
      const float gw = 2.f * (-qz * GRq[1] + qy * GRq[2] + qz * GRq[3] - qx * GRq[5] - qy * GRq[6] + qx * GRq[7]);
      const float gx = 2.f * (qy * GRq[1] + qz * GRq[2] + qy * GRq[3] - 2.f * qx * GRq[4] - qw * GRq[5] + qz * GRq[6] +
                              qw * GRq[7] - 2.f * qx * GRq[8]);
      const float gy = 2.f * (-2.f * qy * GRq[0] + qx * GRq[1] + qw * GRq[2] + qx * GRq[3] + qz * GRq[5] - qw * GRq[6] +
                              qz * GRq[7] - 2.f * qy * GRq[8]);
      const float gzq = 2.f * (-2.f * qz * GRq[0] - qw * GRq[1] + qx * GRq[2] + qw * GRq[3] - 2.f * qz * GRq[4] +
                               qy * GRq[5] + qx * GRq[6] + qy * GRq[7]);
      const float dot = gw * qw + gx * qx + gy * qy + gzq * qz;
      // q^ = q / |q| (R18)
      const float4 gq = make_float4((gw - qw * dot) * iq, (gx - qx * dot) * iq, (gy - qy * dot) * iq, (gzq - qz * dot) * iq);
      float4 m = a.g_mean_opa[i];
      a.g_mean_opa[i] = make_float4(m.x + gmu[0], m.y + gmu[1], m.z + gmu[2], m.w + gb.z);
      float4 qq = a.g_quat[i];
      a.g_quat[i] = make_float4(qq.x + gq.x, qq.y + gq.y, qq.z + gq.z, qq.w + gq.w);
      float4 l = a.g_logscale[i];
      a.g_logscale[i] = make_float4(l.x + gls[0], l.y + gls[1], l.z + gls[2], l.w);
      float4 cc = a.g_rgb[i];
      a.g_rgb[i] = make_float4(cc.x + gc.x, cc.y + gc.y, cc.z + gc.z, cc.w);
    }
    if (kPose) {
      // dL/dt = dL/dp; dL/dR = dL/dp mu^T + 2 G_Sc R Sigma
      float RS[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) RS[3 * r + c] = R[3 * r] * Sig[c] + R[3 * r + 1] * Sig[3 + c] + R[3 * r + 2] * Sig[6 + c];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          pose[3 * r + c] =
              gp[r] * mu[c] + 2.f * (GSc[3 * r] * RS[c] + GSc[3 * r + 1] * RS[3 + c] + GSc[3 * r + 2] * RS[6 + c]);
#pragma unroll
      for (int k = 0; k < 3; ++k) pose[9 + k] = gp[k];
    }
  }
  if (kPose) {
    // fixed-order block reduction: warp shuffles, then warp partials summed by thread order
    __shared__ float sh[8][12];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      float v = pose[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < 12) {
      float v = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sh[w][threadIdx.x];
      a.pose_partials[size_t(blockIdx.x) * 12 + threadIdx.x] = v;
    }
  }
}

}  // namespace gs

extern "C" size_t gs_bwd_workspace_bytes(int32_t n) {
  if (n < 0) return 0;
  return size_t(n > 0 ? n : 1) * gs::kG2 * sizeof(float);
}

extern "C" int32_t gs_pose_partials_count(int32_t n) {
  if (n < 0) return 0;
  return n > 0 ? (n + 255) / 256 : 1;
}

extern "C" int gs_render_bwd(gs_params p, const gs_view *view, gs_camera cam, gs_proj pr, const int32_t *sorted_idx,
                             const int32_t *tile_range, const float *T_final, const int32_t *n_contrib,
                             const float *dL_dcolor, const float *dL_ddepth, const float *dL_dalpha, uint32_t flags,
                             void *ws, size_t ws_bytes, float *g_mean_opa, float *g_quat, float *g_logscale,
                             float *g_rgb, float *pose_partials, void *stream) {
  using namespace gs;
  const bool want_params = flags & GS_GRAD_PARAMS, want_pose = flags & GS_GRAD_POSE;
  const bool run_pixels = !(flags & GS_BWD_GAUSS_ONLY), run_gauss = !(flags & GS_BWD_PIXELS_ONLY);
  if (p.n < 0 || !view || !camera_ok(cam) || !tile_range || !T_final || !n_contrib || !dL_dcolor || !dL_ddepth ||
      (flags & ~(GS_GRAD_PARAMS | GS_GRAD_POSE | GS_BWD_PIXELS_ONLY | GS_BWD_GAUSS_ONLY)) ||
      !(want_params || want_pose) || !(run_pixels || run_gauss)) {
    set_error("gs_render_bwd: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (want_params && (!g_mean_opa || !g_quat || !g_logscale || !g_rgb || !aligned16(g_mean_opa) ||
                      !aligned16(g_quat) || !aligned16(g_logscale) || !aligned16(g_rgb))) {
    set_error("gs_render_bwd: GS_GRAD_PARAMS needs four aligned gradient arrays");
    return GS_ERR_INVALID_ARG;
  }
  if (want_pose && !pose_partials) {
    set_error("gs_render_bwd: GS_GRAD_POSE needs pose_partials");
    return GS_ERR_INVALID_ARG;
  }
  if (p.n > 0) {
    const void *ptrs[] = {p.mean_opa, p.quat, p.logscale, pr.uv, pr.coef, pr.rgbz, pr.conic_o};
    for (const void *x : ptrs)
      if (!x || !aligned16(x)) {
        set_error("gs_render_bwd: null or misaligned parameter/projection array");
        return GS_ERR_INVALID_ARG;
      }
    if (!pr.tiles_touched) {
      set_error("gs_render_bwd: null tiles_touched");
      return GS_ERR_INVALID_ARG;
    }
  }
  if (!ws || ws_bytes < gs_bwd_workspace_bytes(p.n) || !aligned16(ws)) {
    set_error("gs_render_bwd: workspace too small or misaligned");
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  float *grad2d = static_cast<float *>(ws);
  if (p.n == 0) return GS_OK;
  BwdArgs b{reinterpret_cast<const double2 *>(pr.uv), reinterpret_cast<const float4 *>(pr.coef),
            reinterpret_cast<const float4 *>(pr.rgbz), reinterpret_cast<const float4 *>(pr.conic_o), sorted_idx,
            reinterpret_cast<const int2 *>(tile_range), T_final, n_contrib, dL_dcolor, dL_ddepth, dL_dalpha,
            cam.width, cam.height, tiles_x(cam), grad2d};
  const int T = tiles_x(cam) * tiles_y(cam);
  if (run_pixels) {
    if (want_params)
      k_bwd_pixels<true><<<T, kTilePx, 0, s>>>(b);
    else
      k_bwd_pixels<false><<<T, kTilePx, 0, s>>>(b);
  }
  if (!run_gauss) return check_launch("gs_render_bwd");
  GaussArgs g{p, view, cam.fx, cam.fy, reinterpret_cast<const float4 *>(pr.conic_o), pr.tiles_touched, grad2d,
              reinterpret_cast<float4 *>(g_mean_opa), reinterpret_cast<float4 *>(g_quat),
              reinterpret_cast<float4 *>(g_logscale), reinterpret_cast<float4 *>(g_rgb), pose_partials};
  const int blocks = gs_pose_partials_count(p.n);
  if (want_params && want_pose)
    k_bwd_gauss<true, true><<<blocks, 256, 0, s>>>(g);
  else if (want_params)
    k_bwd_gauss<true, false><<<blocks, 256, 0, s>>>(g);
  else
    k_bwd_gauss<false, true><<<blocks, 256, 0, s>>>(g);
  return check_launch("gs_render_bwd");
}
