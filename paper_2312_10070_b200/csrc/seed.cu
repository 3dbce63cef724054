// seed.cu — NEXT(4) gs_seed: sub-map seeding from a keyframe (P:155-156,
// P:230; R37-R41).
//
//   1. candidates: the first M_k pixels with valid depth and rendered alpha
//      < alpha_n, in the order of a seeded bijective permutation of the pixel
//      indices (R37, R38) — a stream compaction over the permuted order;
//   2. back-projection in fp64, rounded to the stored fp32 means (R39);
//   3. a uniform grid (cell 0.1 m, open-addressing hash of the cell) over the
//      existing means and the candidates; a candidate is rejected if an
//      existing mean or an earlier candidate lies within rho (R40);
//   4. every accepted point becomes a Gaussian appended after the n existing
//      ones: colour of its pixel, opacity 0.5, identity rotation, log-scales
//      ln(clamp(nearest-neighbour distance among the existing means and the
//      accepted points, rho / 2, 0.1 m)) (R41).
// Distances are fp64 on the fp32 points, compared squared; the grid only
// prunes the brute-force search (points within 0.1 m lie in adjacent cells).
// Compactions are block counts + one-CTA scan + ballot scatter: the output
// order is deterministic (sample order).
//
// gs_gradient_mask (the first keyframe's M_c batch, R43): the grey image's
// squared Sobel magnitude in fp64 (the oracle's operation order, no
// contraction), its exact nearest-rank percentile by an 8-pass MSB radix
// select over the fp64 bit patterns, and a pseudo-alpha map (0 on the
// high-gradient valid-depth pixels, 1 elsewhere) that gs_seed's alpha gate
// turns into that candidate set.
#include <algorithm>
#include <cmath>

#include "gs_internal.cuh"

namespace gs {

constexpr int kSdThreads = 256;
constexpr double kCell = 0.1;  // NN grid cell = the NN clamp (R41); the rejection grid uses cells of rho
constexpr uint64_t kEmpty = 0ull;

struct SeedLayout {
  size_t bcount, bacc, misc, perm_cand, pts, keys, cnt, start, fill, items, acc, nn, total;
  int nblk_pix, nblk_cand, nblk_slot;
  uint32_t ts;  // hash-table slots (power of two)
};

static SeedLayout seed_layout(int64_t HW, int32_t n, int32_t max_new) {
  SeedLayout L;
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off = (off + b + 255) & ~size_t(255);
    return o;
  };
  L.nblk_pix = int(std::max<int64_t>(1, (HW + kSdThreads - 1) / kSdThreads));
  L.nblk_cand = std::max(1, (max_new + kSdThreads - 1) / kSdThreads);
  uint32_t ts = 1024;
  while (ts < 2u * uint32_t(n + max_new)) ts <<= 1;
  L.ts = ts;
  L.nblk_slot = int((ts + kSdThreads - 1) / kSdThreads);
  const int nb = std::max(L.nblk_pix, std::max(L.nblk_cand, L.nblk_slot));
  L.bcount = take(4 * size_t(nb + 1));
  L.bacc = take(4 * size_t(L.nblk_cand + 1));
  L.misc = take(64);  // [0] K candidates, [1] accepted
  L.perm_cand = take(4 * size_t(std::max(max_new, 1)));
  L.pts = take(12 * size_t(std::max(max_new, 1)));
  L.keys = take(8 * size_t(ts));
  L.cnt = take(4 * size_t(ts));
  L.start = take(4 * size_t(ts));
  L.fill = take(4 * size_t(ts));
  L.items = take(4 * size_t(n + std::max(max_new, 1)));
  L.acc = take(4 * size_t(std::max(max_new, 1)));
  L.nn = take(8 * size_t(std::max(max_new, 1)));
  L.total = off;
  return L;
}

// ---- R38: the seeded bijection of [0, n) ------------------------------------------
__device__ __forceinline__ uint64_t perm_round(uint64_t x, uint64_t s, uint64_t mask, int half) {
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    x = (x ^ ((s + 0x9E3779B9ull * uint64_t(r + 1)) & mask)) & mask;
    x = (x * 0x2545F491ull) & mask;
    x = x ^ (x >> half);
  }
  return x;
}

__device__ __forceinline__ int perm_index(int i, int n, uint32_t seed, int m) {
  const uint64_t mask = (uint64_t(1) << m) - 1;
  uint64_t x = perm_round(uint64_t(i), seed, mask, (m + 1) / 2);
  while (x >= uint64_t(n)) x = perm_round(x, seed, mask, (m + 1) / 2);  // cycle-walking
  return int(x);
}

// ---- compaction helpers ----------------------------------------------------------
__device__ __forceinline__ void block_count_store(bool flag, int *bcount) {
  __shared__ int sh[kSdThreads / 32];
  const int c = __popc(__ballot_sync(0xffffffffu, flag));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kSdThreads / 32; ++w) s += sh[w];
    bcount[blockIdx.x] = s;
  }
}

// in-place exclusive scan of nblk counts (one CTA); total -> *total
__global__ void __launch_bounds__(1024) k_sd_scan(int *bcount, const int *nblk_dev, int nblk_host, int *total) {
  __shared__ int sh[1024];
  __shared__ int carry;
  const int nblk = nblk_dev ? min(*nblk_dev, nblk_host) : nblk_host;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblk; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const int v = b < nblk ? bcount[b] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int y = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += y;
      __syncthreads();
    }
    if (b < nblk) bcount[b] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// rank of a flagged element = its block offset + the flagged elements before it in the block
__device__ __forceinline__ int block_rank(bool flag, const int *boff) {
  __shared__ int sh[kSdThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) sh[w] = __popc(b);
  __syncthreads();
  int r = boff[blockIdx.x];
  for (int ww = 0; ww < w; ++ww) r += sh[ww];
  return r + __popc(b & lanemask_lt());
}

struct SeedArgs {
  const float *color, *depth, *alpha;
  int W, H, HW, m;
  uint32_t seed;
  float alpha_n;
  double fx, fy, cx, cy, R[9], t[3];
  const float4 *means;  // existing [n] (mean_opa)
  int n, max_new;
  double rho2, rho;
  uint32_t ts;
  double cell;  // cell size of the grid being built / queried
  int accepted_only;  // grid over the existing means + accepted candidates (else all candidates)
  int *bcount, *bacc, *misc, *cand;  // bacc: block offsets of the accepted; misc[0] = K, misc[1] = accepted
  float *pts;                 // [K][3]
  uint64_t *keys;
  int *cnt, *start, *fill, *items, *acc;
  double *nn;  // [K] squared nearest-neighbour distances of the accepted points
  float4 *o_mean_opa, *o_quat, *o_logscale, *o_rgb;  // written at [n + rank]
  int capacity;
};

__device__ __forceinline__ bool eligible(const SeedArgs &a, int p) {
  return __ldg(a.depth + p) > 0.f && __ldg(a.alpha + p) < a.alpha_n;  // R37
}

__global__ void __launch_bounds__(kSdThreads) k_sd_count(SeedArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  block_count_store(i < a.HW && eligible(a, perm_index(i, a.HW, a.seed, a.m)), a.bcount);
}

__global__ void __launch_bounds__(kSdThreads) k_sd_select(SeedArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = i < a.HW ? perm_index(i, a.HW, a.seed, a.m) : 0;
  const bool e = i < a.HW && eligible(a, p);
  const int r = block_rank(e, a.bcount);
  if (e && r < a.max_new) a.cand[r] = p;
}

// misc[0] = the eligible total from the scan -> K = min(total, max_new)
__global__ void k_sd_clampK(int *misc, int max_new) {
  misc[0] = min(misc[0], max_new);
}

// R39: p_c = ((i - cx) D / fx, (j - cy) D / fy, D); world = R^T (p_c - t)
__global__ void __launch_bounds__(kSdThreads) k_sd_points(SeedArgs a) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.misc[0]) return;
  const int p = a.cand[k];
  const double i = double(p % a.W), j = double(p / a.W), z = double(__ldg(a.depth + p));
  const double pc[3] = {__dmul_rn(__dsub_rn(i, a.cx), z) / a.fx, __dmul_rn(__dsub_rn(j, a.cy), z) / a.fy, z};
  const double d[3] = {__dsub_rn(pc[0], a.t[0]), __dsub_rn(pc[1], a.t[1]), __dsub_rn(pc[2], a.t[2])};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    // (R^T d)_c = sum_r R[r][c] d_r, summed in row order (as the oracle's matmul)
    const double w = __dadd_rn(__dadd_rn(__dmul_rn(d[0], a.R[c]), __dmul_rn(d[1], a.R[3 + c])), __dmul_rn(d[2], a.R[6 + c]));
    a.pts[3 * k + c] = float(w);
  }
}

__device__ __forceinline__ void point_of(const SeedArgs &a, int id, double q[3]) {
  if (id < a.n) {
    const float4 m = __ldg(a.means + id);
    q[0] = m.x;
    q[1] = m.y;
    q[2] = m.z;
  } else {
    const float *p = a.pts + 3 * (id - a.n);
    q[0] = p[0];
    q[1] = p[1];
    q[2] = p[2];
  }
}

__device__ __forceinline__ uint64_t cell_key(int cx, int cy, int cz) {
  // 21 bits per axis (offset), +1 so that 0 stays the empty key
  return ((uint64_t(cx + (1 << 20)) & 0x1fffff) | ((uint64_t(cy + (1 << 20)) & 0x1fffff) << 21) |
          ((uint64_t(cz + (1 << 20)) & 0x1fffff) << 42)) + 1ull;
}

__device__ __forceinline__ void cell_of(const double q[3], double cell, int c[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k] = int(floor(q[k] / cell));
}

// points of the grid: existing means, then candidates (all, or accepted only)
__device__ __forceinline__ bool in_grid(const SeedArgs &a, int id) {
  return id < a.n || (id < a.n + a.misc[0] && (!a.accepted_only || a.acc[id - a.n]));
}

__device__ __forceinline__ uint32_t slot_hash(uint64_t key, uint32_t ts) {
  key ^= key >> 33;
  key *= 0xff51afd7ed558ccdull;
  key ^= key >> 33;
  return uint32_t(key) & (ts - 1);
}

// insert-or-find (insert = true) / find (returns -1 if absent)
__device__ int slot_of(const SeedArgs &a, uint64_t key, bool insert) {
  uint32_t s = slot_hash(key, a.ts);
  while (true) {
    const uint64_t k = insert ? atomicCAS(reinterpret_cast<unsigned long long *>(a.keys + s), kEmpty, key)
                              : a.keys[s];
    if (k == key || (insert && k == kEmpty)) return int(s);
    if (!insert && k == kEmpty) return -1;
    s = (s + 1) & (a.ts - 1);
  }
}

__global__ void __launch_bounds__(kSdThreads) k_sd_grid_count(SeedArgs a) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (!in_grid(a, id)) return;
  double q[3];
  int c[3];
  point_of(a, id, q);
  cell_of(q, a.cell, c);
  atomicAdd(a.cnt + slot_of(a, cell_key(c[0], c[1], c[2]), true), 1);
}

// exclusive scan of the slot counts in blocks of kSdThreads: block sums ...
__global__ void __launch_bounds__(kSdThreads) k_sd_slot_sums(SeedArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = s < int(a.ts) ? a.cnt[s] : 0;
  __shared__ int sh[kSdThreads / 32];
  int x = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kSdThreads / 32; ++w) t += sh[w];
    a.bcount[blockIdx.x] = t;
  }
}

// ... then per slot: block offset + the counts before it in the block
__global__ void __launch_bounds__(kSdThreads) k_sd_slot_start(SeedArgs a) {
  __shared__ int sh[kSdThreads];
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = s < int(a.ts) ? a.cnt[s] : 0;
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = 1; o < kSdThreads; o <<= 1) {
    const int y = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += y;
    __syncthreads();
  }
  if (s < int(a.ts)) a.start[s] = a.bcount[blockIdx.x] + sh[threadIdx.x] - v;
}

__global__ void __launch_bounds__(kSdThreads) k_sd_grid_fill(SeedArgs a) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (!in_grid(a, id)) return;
  double q[3];
  int c[3];
  point_of(a, id, q);
  cell_of(q, a.cell, c);
  const int s = slot_of(a, cell_key(c[0], c[1], c[2]), false);
  a.items[a.start[s] + atomicAdd(a.fill + s, 1)] = id;
}

__device__ __forceinline__ double dist2(const double o[3], const double q[3]) {
  return __dadd_rn(__dadd_rn(__dmul_rn(o[0] - q[0], o[0] - q[0]), __dmul_rn(o[1] - q[1], o[1] - q[1])),
                   __dmul_rn(o[2] - q[2], o[2] - q[2]));
}

// R40: rejected if an existing mean, or an earlier candidate, is within rho.
// One warp per candidate: lanes 0..26 take one neighbouring cell each.
__global__ void __launch_bounds__(kSdThreads) k_sd_reject(SeedArgs a) {
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= a.misc[0]) return;
  double q[3];
  int c[3];
  point_of(a, a.n + k, q);
  cell_of(q, a.cell, c);
  bool hit = false;
  if (lane < 27) {
    const int s = slot_of(a, cell_key(c[0] + lane % 3 - 1, c[1] + (lane / 3) % 3 - 1, c[2] + lane / 9 - 1), false);
    if (s >= 0)
      for (int e = a.start[s], e1 = e + a.cnt[s]; e < e1 && !hit; ++e) {
        const int id = a.items[e];
        if (id >= a.n && id - a.n >= k) continue;  // only earlier candidates
        double o[3];
        point_of(a, id, o);
        hit = dist2(o, q) < a.rho2;
      }
  }
  if (lane == 0) a.acc[k] = !__any_sync(0xffffffffu, hit);
  else __any_sync(0xffffffffu, hit);
}

__global__ void __launch_bounds__(kSdThreads) k_sd_acc_count(SeedArgs a) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  block_count_store(k < a.misc[0] && a.acc[k], a.bacc);
}

// R41: the nearest-neighbour distance of accepted point k (one warp, lanes
// over the 27 cells of the 0.1 m grid of existing + accepted points)
__global__ void __launch_bounds__(kSdThreads) k_sd_nn(SeedArgs a) {
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= a.misc[0] || !a.acc[k]) return;
  double q[3];
  int c[3];
  point_of(a, a.n + k, q);
  cell_of(q, a.cell, c);
  double best = INFINITY;
  if (lane < 27) {
    const int s = slot_of(a, cell_key(c[0] + lane % 3 - 1, c[1] + (lane / 3) % 3 - 1, c[2] + lane / 9 - 1), false);
    if (s >= 0)
      for (int e = a.start[s], e1 = e + a.cnt[s]; e < e1; ++e) {
        const int id = a.items[e];
        if (id == a.n + k) continue;  // itself (the grid holds existing + accepted points only)
        double o[3];
        point_of(a, id, o);
        best = fmin(best, dist2(o, q));
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) a.nn[k] = best;
}

// R41: accepted points -> Gaussians at [n + rank] (sample order)
__global__ void __launch_bounds__(kSdThreads) k_sd_emit(SeedArgs a) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = k < a.misc[0] && a.acc[k];
  const int r = block_rank(ok, a.bacc);
  if (!ok || a.n + r >= a.capacity) return;
  double q[3];
  point_of(a, a.n + k, q);
  // neighbours beyond 0.1 m may be missed by the 27 cells: the clamp makes them irrelevant
  const double d = fmin(fmax(sqrt(a.nn[k]), a.rho * 0.5), kCell);
  const float ls = float(log(d));
  const int o = a.n + r;
  const int p = a.cand[k];
  a.o_mean_opa[o] = make_float4(float(q[0]), float(q[1]), float(q[2]), 0.f);  // opacity 0.5
  a.o_quat[o] = make_float4(1.f, 0.f, 0.f, 0.f);
  a.o_logscale[o] = make_float4(ls, ls, ls, 0.f);
  a.o_rgb[o] = make_float4(__ldg(a.color + p), __ldg(a.color + a.HW + p), __ldg(a.color + 2 * a.HW + p), 0.f);
}

// ---- R43: high-colour-gradient mask --------------------------------------------
constexpr int kGmThreads = 256;

__global__ void __launch_bounds__(kGmThreads) k_gm_grey(const float *__restrict__ color, int64_t HW, double *grey) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= HW) return;
  const double r = __ldg(color + q), g = __ldg(color + HW + q), b = __ldg(color + 2 * HW + q);
  grey[q] = __dadd_rn(__dadd_rn(__dmul_rn(0.299, r), __dmul_rn(0.587, g)), __dmul_rn(0.114, b));
}

__global__ void __launch_bounds__(kGmThreads) k_gm_m2(const double *__restrict__ grey, int W, int H,
                                                      uint64_t *keys) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= int64_t(W) * H) return;
  const int i = int(q % W), j = int(q / W);
  double m2 = 0.0;
  if (i > 0 && j > 0 && i < W - 1 && j < H - 1) {
    auto G = [&](int y, int x) { return grey[int64_t(y) * W + x]; };
    // gx = right - left column, gy = bottom - top row, weights (1, 2, 1), the oracle's order
    const double gx = __dsub_rn(__dadd_rn(__dadd_rn(G(j - 1, i + 1), __dmul_rn(2.0, G(j, i + 1))), G(j + 1, i + 1)),
                                __dadd_rn(__dadd_rn(G(j - 1, i - 1), __dmul_rn(2.0, G(j, i - 1))), G(j + 1, i - 1)));
    const double gy = __dsub_rn(__dadd_rn(__dadd_rn(G(j + 1, i - 1), __dmul_rn(2.0, G(j + 1, i))), G(j + 1, i + 1)),
                                __dadd_rn(__dadd_rn(G(j - 1, i - 1), __dmul_rn(2.0, G(j - 1, i))), G(j - 1, i + 1)));
    m2 = __dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy));
  }
  keys[q] = uint64_t(__double_as_longlong(m2));  // m2 >= +0: bit order = value order
}

// select state: [0] prefix of the k-th key, [1] k (1-based rank among the
// keys matching the prefix); hist [256]
__global__ void __launch_bounds__(kGmThreads) k_gm_hist(const uint64_t *__restrict__ keys, int64_t HW, int shift,
                                                        const unsigned long long *state, unsigned *hist) {
  __shared__ unsigned sh[256];
  sh[threadIdx.x] = 0u;
  __syncthreads();
  const uint64_t prefix = state[0];
  const uint64_t hi_mask = shift >= 56 ? 0ull : ~((uint64_t(1) << (shift + 8)) - 1);
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < HW; q += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[q];
    if ((k & hi_mask) == (prefix & hi_mask)) atomicAdd(&sh[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_gm_pick(int shift, unsigned long long *state, unsigned *hist) {
  __shared__ unsigned sh[256];
  const unsigned c = hist[threadIdx.x];
  sh[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {  // the digit whose cumulative count reaches k (fixed order)
    unsigned long long k = state[1], cum = 0;
    int d = 0;
    for (; d < 255; ++d) {
      if (cum + sh[d] >= k) break;
      cum += sh[d];
    }
    state[0] |= (unsigned long long)d << shift;
    state[1] = k - cum;
  }
  hist[threadIdx.x] = 0u;  // for the next pass
}

__global__ void __launch_bounds__(256) k_gm_init(unsigned long long *state, unsigned *hist, unsigned long long k) {
  if (threadIdx.x == 0) {
    state[0] = 0ull;
    state[1] = k;
  }
  hist[threadIdx.x] = 0u;
}

__global__ void __launch_bounds__(kGmThreads) k_gm_mask(const uint64_t *__restrict__ keys,
                                                        const float *__restrict__ depth, int64_t HW,
                                                        const unsigned long long *state, float *pseudo_alpha) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= HW) return;
  pseudo_alpha[q] = (keys[q] > state[0] && __ldg(depth + q) > 0.f) ? 0.f : 1.f;
}

}  // namespace gs

extern "C" size_t gs_gradient_mask_workspace_bytes(gs_camera cam) {
  if (!gs::camera_ok(cam)) return 0;
  return 16 * size_t(cam.width) * cam.height + 2048;  // grey + keys (fp64 / uint64 per pixel), state, histogram
}

extern "C" int gs_gradient_mask(gs_camera cam, const float *color, const float *depth, double q, float *pseudo_alpha,
                                double *threshold_m2, void *ws, size_t ws_bytes, void *stream) {
  using namespace gs;
  if (!camera_ok(cam) || !color || !depth || !pseudo_alpha || !(q > 0.0 && q <= 1.0)) {
    set_error("gs_gradient_mask: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  const int64_t HW = int64_t(cam.width) * cam.height;
  if (!ws || ws_bytes < gs_gradient_mask_workspace_bytes(cam) || (reinterpret_cast<uintptr_t>(ws) & 7u)) {
    set_error("gs_gradient_mask: workspace too small or misaligned");
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char *w = static_cast<char *>(ws);
  double *grey = reinterpret_cast<double *>(w);
  uint64_t *keys = reinterpret_cast<uint64_t *>(w + 8 * size_t(HW));
  unsigned long long *state = reinterpret_cast<unsigned long long *>(w + 16 * size_t(HW));
  unsigned *hist = reinterpret_cast<unsigned *>(w + 16 * size_t(HW) + 64);
  // nearest rank: the ceil(q HW)-th smallest (fp64 product, as the oracle)
  const unsigned long long k = (unsigned long long)std::max<double>(1.0, std::ceil(q * double(HW)));
  k_gm_init<<<1, 256, 0, s>>>(state, hist, k);
  const int nb = int((HW + kGmThreads - 1) / kGmThreads);
  k_gm_grey<<<nb, kGmThreads, 0, s>>>(color, HW, grey);
  k_gm_m2<<<nb, kGmThreads, 0, s>>>(grey, cam.width, cam.height, keys);
  const int nh = std::min(nb, 148 * 8);
  for (int shift = 56; shift >= 0; shift -= 8) {
    k_gm_hist<<<nh, kGmThreads, 0, s>>>(keys, HW, shift, state, hist);
    k_gm_pick<<<1, 256, 0, s>>>(shift, state, hist);
  }
  k_gm_mask<<<nb, kGmThreads, 0, s>>>(keys, depth, HW, state, pseudo_alpha);
  if (threshold_m2) cudaMemcpyAsync(threshold_m2, state, sizeof(double), cudaMemcpyDeviceToDevice, s);
  return check_launch("gs_gradient_mask");
}

extern "C" size_t gs_seed_workspace_bytes(gs_camera cam, int32_t n, int32_t max_new) {
  if (!gs::camera_ok(cam) || n < 0 || max_new < 0) return 0;
  return gs::seed_layout(int64_t(cam.width) * cam.height, n, max_new).total;
}

extern "C" int gs_seed(gs_camera cam, const gs_view *view_host, const float *color, const float *depth,
                       const float *alpha, float alpha_n, float rho, int32_t max_new, uint32_t seed, gs_params p,
                       int32_t capacity, void *ws, size_t ws_bytes, int32_t *n_new, void *stream) {
  using namespace gs;
  if (max_new == 0 && n_new && camera_ok(cam)) {  // nothing to seed
    cudaMemsetAsync(n_new, 0, sizeof(int32_t), as_stream(stream));
    return check_launch("gs_seed");
  }
  if (!camera_ok(cam) || !view_host || !color || !depth || !alpha || !n_new || max_new < 0 || p.n < 0 ||
      capacity < p.n || !(rho > 0.f && rho <= float(kCell)) || (p.n > 0 && !p.mean_opa) || !p.quat ||
      !p.logscale || !p.rgb || !p.mean_opa) {
    set_error("gs_seed: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  const int64_t HW = int64_t(cam.width) * cam.height;
  const SeedLayout L = seed_layout(HW, p.n, max_new);
  if (!ws || ws_bytes < L.total) {
    set_error("gs_seed: workspace %zu < %zu bytes", ws_bytes, L.total);
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char *w = static_cast<char *>(ws);
  SeedArgs a;
  a.color = color;
  a.depth = depth;
  a.alpha = alpha;
  a.W = cam.width;
  a.H = cam.height;
  a.HW = int(HW);
  int m = 1;
  while ((int64_t(1) << m) < std::max<int64_t>(HW, 2)) ++m;
  a.m = m;
  a.seed = seed;
  a.alpha_n = alpha_n;
  a.fx = cam.fx;
  a.fy = cam.fy;
  a.cx = cam.cx;
  a.cy = cam.cy;
  for (int k = 0; k < 9; ++k) a.R[k] = view_host->R[k];
  for (int k = 0; k < 3; ++k) a.t[k] = view_host->t[k];
  a.means = reinterpret_cast<const float4 *>(p.mean_opa);
  a.n = p.n;
  a.max_new = max_new;
  a.rho = double(rho);
  a.rho2 = double(rho) * double(rho);
  a.ts = L.ts;
  a.bcount = reinterpret_cast<int *>(w + L.bcount);
  a.bacc = reinterpret_cast<int *>(w + L.bacc);
  a.misc = reinterpret_cast<int *>(w + L.misc);
  a.cand = reinterpret_cast<int *>(w + L.perm_cand);
  a.pts = reinterpret_cast<float *>(w + L.pts);
  a.keys = reinterpret_cast<uint64_t *>(w + L.keys);
  a.cnt = reinterpret_cast<int *>(w + L.cnt);
  a.start = reinterpret_cast<int *>(w + L.start);
  a.fill = reinterpret_cast<int *>(w + L.fill);
  a.items = reinterpret_cast<int *>(w + L.items);
  a.acc = reinterpret_cast<int *>(w + L.acc);
  a.nn = reinterpret_cast<double *>(w + L.nn);
  a.o_mean_opa = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.mean_opa));
  a.o_quat = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.quat));
  a.o_logscale = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.logscale));
  a.o_rgb = const_cast<float4 *>(reinterpret_cast<const float4 *>(p.rgb));
  a.capacity = capacity;
  // 1. candidates in permuted order
  k_sd_count<<<L.nblk_pix, kSdThreads, 0, s>>>(a);
  k_sd_scan<<<1, 1024, 0, s>>>(a.bcount, nullptr, L.nblk_pix, a.misc + 0);
  k_sd_select<<<L.nblk_pix, kSdThreads, 0, s>>>(a);
  k_sd_clampK<<<1, 1, 0, s>>>(a.misc, max_new);
  // 2. points
  k_sd_points<<<L.nblk_cand, kSdThreads, 0, s>>>(a);
  // 3. a grid of rho cells over existing means + all candidates -> rejection;
  // 4. a grid of 0.1 m cells over existing means + accepted points -> NN scales
  const int nb_pts = std::max(1, (p.n + max_new + kSdThreads - 1) / kSdThreads);
  auto build = [&](double cell, int accepted_only) {
    a.cell = cell;
    a.accepted_only = accepted_only;
    cudaMemsetAsync(w + L.keys, 0, 8 * size_t(L.ts), s);
    cudaMemsetAsync(w + L.cnt, 0, 4 * size_t(L.ts), s);
    cudaMemsetAsync(w + L.fill, 0, 4 * size_t(L.ts), s);
    k_sd_grid_count<<<nb_pts, kSdThreads, 0, s>>>(a);
    k_sd_slot_sums<<<L.nblk_slot, kSdThreads, 0, s>>>(a);
    k_sd_scan<<<1, 1024, 0, s>>>(a.bcount, nullptr, L.nblk_slot, a.misc + 2);
    k_sd_slot_start<<<L.nblk_slot, kSdThreads, 0, s>>>(a);
    k_sd_grid_fill<<<nb_pts, kSdThreads, 0, s>>>(a);
  };
  const int nb_warp = std::max(1, (max_new + kSdThreads / 32 - 1) / (kSdThreads / 32));
  build(double(rho), 0);
  k_sd_reject<<<nb_warp, kSdThreads, 0, s>>>(a);
  k_sd_acc_count<<<L.nblk_cand, kSdThreads, 0, s>>>(a);
  k_sd_scan<<<1, 1024, 0, s>>>(a.bacc, nullptr, L.nblk_cand, a.misc + 1);
  build(kCell, 1);
  k_sd_nn<<<nb_warp, kSdThreads, 0, s>>>(a);
  k_sd_emit<<<L.nblk_cand, kSdThreads, 0, s>>>(a);
  cudaMemcpyAsync(n_new, a.misc + 1, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
  return check_launch("gs_seed");
}
