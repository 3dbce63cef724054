// pose.cu — S7 gs_pose_grad: camera-pose gradient for frame-to-model tracking
// (Eq. 14; R22) and an optional device-side Adam step on the
// left-perturbation twist, so a tracking iteration needs no host
// round trip and can be captured in a CUDA graph.
//
// One CTA: the pose partials of gs_render_bwd are summed in fp64 in a fixed
// order (lane l takes records l, l+64, ... in order; then a fixed pairwise tree
// over the lanes), so the result is bit-deterministic.
#include "gs_internal.cuh"

namespace gs {

__device__ void quat_to_rot_d(const double *q, double *R) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
}

// Shepperd's method, unit quaternion (w, x, y, z) with w >= 0.
__device__ void rot_to_quat_d(const double *R, double *q) {
  const double tr = R[0] + R[4] + R[8];
  double w, x, y, z;
  if (tr > 0.0) {
    const double s = 2.0 * sqrt(tr + 1.0);
    w = 0.25 * s;
    x = (R[7] - R[5]) / s;
    y = (R[2] - R[6]) / s;
    z = (R[3] - R[1]) / s;
  } else if (R[0] > R[4] && R[0] > R[8]) {
    const double s = 2.0 * sqrt(1.0 + R[0] - R[4] - R[8]);
    w = (R[7] - R[5]) / s;
    x = 0.25 * s;
    y = (R[1] + R[3]) / s;
    z = (R[2] + R[6]) / s;
  } else if (R[4] > R[8]) {
    const double s = 2.0 * sqrt(1.0 + R[4] - R[0] - R[8]);
    w = (R[2] - R[6]) / s;
    x = (R[1] + R[3]) / s;
    y = 0.25 * s;
    z = (R[5] + R[7]) / s;
  } else {
    const double s = 2.0 * sqrt(1.0 + R[8] - R[0] - R[4]);
    w = (R[3] - R[1]) / s;
    x = (R[2] + R[6]) / s;
    y = (R[5] + R[7]) / s;
    z = 0.25 * s;
  }
  double n = sqrt(w * w + x * x + y * y + z * z);
  if (w < 0.0) n = -n;
  q[0] = w / n;
  q[1] = x / n;
  q[2] = y / n;
  q[3] = z / n;
}

// SE(3) exponential of xi = (v, w): Rodrigues + left Jacobian V.
__device__ void se3_exp_d(const double *xi, double *R, double *t) {
  const double *v = xi, *w = xi + 3;
  const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2], th = sqrt(th2);
  const double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
  double K2[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) K2[3 * a + b] = K[3 * a] * K[b] + K[3 * a + 1] * K[3 + b] + K[3 * a + 2] * K[6 + b];
  double A, B, Cc;
  if (th < 1e-8) {
    A = 1.0 - th2 / 6.0;
    B = 0.5 - th2 / 24.0;
    Cc = 1.0 / 6.0 - th2 / 120.0;
  } else {
    double sn, cs;
    sincos(th, &sn, &cs);
    A = sn / th;
    B = (1.0 - cs) / th2;
    Cc = (th - sn) / (th2 * th);
  }
  double V[9];
  for (int i = 0; i < 9; ++i) {
    const double I = (i % 4 == 0) ? 1.0 : 0.0;
    R[i] = I + A * K[i] + B * K2[i];
    V[i] = I + B * K[i] + Cc * K2[i];
  }
  for (int i = 0; i < 3; ++i) t[i] = V[3 * i] * v[0] + V[3 * i + 1] * v[1] + V[3 * i + 2] * v[2];
}

struct PoseArgs {
  gs_view *view;
  const float *partials;
  int n_partials;
  int has_step;
  gs_pose_step step;
  double *adam;
  float *dL_dview, *dL_dtwist, *dL_dqt;
};

#ifndef POSE_POW
#define POSE_POW 1
#endif
#ifndef POSE_RED
#define POSE_RED 1
#endif
#if POSE_RED
// 64 record lanes x 12 components; the loads of 8 records are issued before
// their (in-order) adds, then a fixed pairwise tree over the lanes
constexpr int kPoseLanes = 64, kPoseThreads = kPoseLanes * 12, kPoseUnroll = 8;
#else
constexpr int kPoseLanes = 32, kPoseThreads = kPoseLanes * 12, kPoseUnroll = 1;
#endif

__global__ void __launch_bounds__(kPoseThreads) k_pose_grad(PoseArgs a) {
  pdl_begin();
  // fixed-order fp64 reduction of the [n][12] partials: thread t owns
  // component c = t % 12 of the records k = t / 12 (mod kPoseLanes) ->
  // consecutive threads read consecutive floats (coalesced); then the lane
  // sums of each component are added in a fixed order
  __shared__ double sh[kPoseLanes][13];
  // the view and the Adam state are fetched now, in the shadow of the reduction
  __shared__ float s_view[12];
  __shared__ double s_adam[13], s_tw[6], s_d[6];
  if (threadIdx.x < 12) s_view[threadIdx.x] = threadIdx.x < 9 ? a.view->R[threadIdx.x] : a.view->t[threadIdx.x - 9];
  if (a.has_step && threadIdx.x >= 32 && threadIdx.x < 45) s_adam[threadIdx.x - 32] = a.adam[threadIdx.x - 32];
  const int c = threadIdx.x % 12, l = threadIdx.x / 12;
  double acc = 0.0;
  int k = l;
  for (; k + (kPoseUnroll - 1) * kPoseLanes < a.n_partials; k += kPoseUnroll * kPoseLanes) {
    float v[kPoseUnroll];
#pragma unroll
    for (int u = 0; u < kPoseUnroll; ++u) v[u] = a.partials[size_t(k + u * kPoseLanes) * 12 + c];
#pragma unroll
    for (int u = 0; u < kPoseUnroll; ++u) acc += double(v[u]);
  }
  for (; k < a.n_partials; k += kPoseLanes) acc += double(a.partials[size_t(k) * 12 + c]);
  sh[l][c] = acc;
  __syncthreads();
#pragma unroll
  for (int st = kPoseLanes / 2; st > 0; st >>= 1) {
    if (l < st) sh[l][c] += sh[l + st][c];
    __syncthreads();
  }
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double gR[9], gt[3], R[9], t[3];
  for (int c = 0; c < 9; ++c) gR[c] = sh[0][c];
  for (int c = 0; c < 3; ++c) gt[c] = sh[0][9 + c];
  for (int c = 0; c < 9; ++c) R[c] = s_view[c];
  for (int c = 0; c < 3; ++c) t[c] = s_view[9 + c];
  // twist of the left perturbation T <- exp(xi^) T:
  // dL/dv = dL/dt, dL/dw_k = <dL/dR, [e_k]x R> + dL/dt . (e_k x t)
  double tw[6];
  for (int k = 0; k < 3; ++k) tw[k] = gt[k];
  {
    // [e_0]x R = rows (0, -R2, R1); [e_1]x R = (R2, 0, -R0); [e_2]x R = (-R1, R0, 0) (rows of R)
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    for (int c = 0; c < 3; ++c) {
      w0 += gR[3 + c] * (-R[6 + c]) + gR[6 + c] * R[3 + c];
      w1 += gR[c] * R[6 + c] + gR[6 + c] * (-R[c]);
      w2 += gR[c] * (-R[3 + c]) + gR[3 + c] * R[c];
    }
    w0 += gt[1] * (-t[2]) + gt[2] * t[1];  // e_0 x t = (0, -t2, t1)
    w1 += gt[0] * t[2] + gt[2] * (-t[0]);  // e_1 x t = (t2, 0, -t0)
    w2 += gt[0] * (-t[1]) + gt[1] * t[0];  // e_2 x t = (-t1, t0, 0)
    tw[3] = w0;
    tw[4] = w1;
    tw[5] = w2;
  }
  if (lane < 6) s_tw[lane] = tw[lane];
  if (a.dL_dview && lane < 12) a.dL_dview[lane] = float(lane < 9 ? gR[lane] : gt[lane - 9]);
  if (a.dL_dtwist && lane < 6) a.dL_dtwist[lane] = float(tw[lane]);
  if (a.dL_dqt && lane == 0) {
    // (q, t) of T_wc: dL/dq = (I - q q^T) sum_ij dL/dR_ij dR_ij/dq
    double q[4];
    rot_to_quat_d(R, q);
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double gw = 2.0 * (-z * gR[1] + y * gR[2] + z * gR[3] - x * gR[5] - y * gR[6] + x * gR[7]);
    const double gx = 2.0 * (y * gR[1] + z * gR[2] + y * gR[3] - 2.0 * x * gR[4] - w * gR[5] + z * gR[6] + w * gR[7] -
                             2.0 * x * gR[8]);
    const double gy = 2.0 * (-2.0 * y * gR[0] + x * gR[1] + w * gR[2] + x * gR[3] + z * gR[5] - w * gR[6] + z * gR[7] -
                             2.0 * y * gR[8]);
    const double gz = 2.0 * (-2.0 * z * gR[0] - w * gR[1] + x * gR[2] + w * gR[3] - 2.0 * z * gR[4] + y * gR[5] +
                             x * gR[6] + y * gR[7]);
    const double dot = gw * w + gx * x + gy * y + gz * z;
    a.dL_dqt[0] = float(gw - w * dot);
    a.dL_dqt[1] = float(gx - x * dot);
    a.dL_dqt[2] = float(gy - y * dot);
    a.dL_dqt[3] = float(gz - z * dot);
    for (int c = 0; c < 3; ++c) a.dL_dqt[4 + c] = float(gt[c]);
  }
  if (a.has_step) {
    // Adam on the twist, applied as T <- exp(d^) T; the six
    // components on six lanes, the retraction on lane 0
    __syncwarp();
    const double b1 = a.step.beta1, b2 = a.step.beta2, eps = a.step.eps;
    const double stp = s_adam[12] + 1.0;
    double d[6];
#if POSE_POW
    // beta^t by binary exponentiation of the integer step (a few ulp from
    // pow; the fp64 pow is a long dependent chain on this single thread)
    double p1 = 1.0, p2 = 1.0, q1 = b1, q2 = b2;
    for (long long e = (long long)stp; e > 0; e >>= 1) {
      if (e & 1) {
        p1 *= q1;
        p2 *= q2;
      }
      q1 *= q1;
      q2 *= q2;
    }
    const double c1 = 1.0 - p1, c2 = 1.0 - p2;  // bias corrections, once
#else
    const double c1 = 1.0 - pow(b1, stp), c2 = 1.0 - pow(b2, stp);  // bias corrections, once
#endif
    if (lane < 6) {
      const int i = lane;
      const double tw_i = s_tw[i];
      const double m = b1 * s_adam[i] + (1.0 - b1) * tw_i;
      const double v = b2 * s_adam[6 + i] + (1.0 - b2) * tw_i * tw_i;
      a.adam[i] = m;
      a.adam[6 + i] = v;
      const double mh = m / c1, vh = v / c2;
      s_d[i] = -(i < 3 ? double(a.step.lr_trans) : double(a.step.lr_rot)) * mh / (sqrt(vh) + eps);
    }
    __syncwarp();
    if (lane != 0) return;
    a.adam[12] = stp;
    for (int i = 0; i < 6; ++i) d[i] = s_d[i];
    double dR[9], dt[3], R2[9], t2[3];
    se3_exp_d(d, dR, dt);
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) R2[3 * r + c] = dR[3 * r] * R[c] + dR[3 * r + 1] * R[3 + c] + dR[3 * r + 2] * R[6 + c];
      t2[r] = dR[3 * r] * t[0] + dR[3 * r + 1] * t[1] + dR[3 * r + 2] * t[2] + dt[r];
    }
    double q[4];
    rot_to_quat_d(R2, q);  // re-orthonormalise through the unit quaternion
    quat_to_rot_d(q, R2);
    for (int c = 0; c < 9; ++c) a.view->R[c] = float(R2[c]);
    for (int c = 0; c < 3; ++c) a.view->t[c] = float(t2[c]);
  }
}

}  // namespace gs

extern "C" int gs_pose_grad(gs_view *view, const float *pose_partials, int32_t n_partials, const gs_pose_step *step,
                            double *adam_state, float *dL_dview, float *dL_dtwist, float *dL_dqt, void *stream) {
  using namespace gs;
  if (!view || !pose_partials || n_partials <= 0 || (step && !adam_state)) {
    set_error("gs_pose_grad: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (step && !(step->lr_trans >= 0.f && step->lr_rot >= 0.f && step->beta1 >= 0.0 && step->beta1 < 1.0 &&
                step->beta2 >= 0.0 && step->beta2 < 1.0 && step->eps > 0.0)) {
    set_error("gs_pose_grad: invalid Adam hyper-parameters");
    return GS_ERR_INVALID_ARG;
  }
  PoseArgs a{view, pose_partials, n_partials, step != nullptr, step ? *step : gs_pose_step{0, 0, 0, 0, 1},
             adam_state, dL_dview, dL_dtwist, dL_dqt};
  launch_pdl(k_pose_grad, dim3(1), dim3(kPoseThreads), 0, as_stream(stream), a);
  return check_launch("gs_pose_grad");
}
