// binsort.cu — S2 gs_bin_sort: tile binning with deterministic depth order
// ("m ordered Gaussians"; R10).
//
// Result = every (tile, Gaussian) pair ordered by the composite key
// (tile asc, fp32 depth asc, Gaussian id asc).  No per-tile sort: the
// visible Gaussians are put in (depth, id) order ONCE, then every tile's list
// is filled by a stable counting pass over that order.
//   1. k_ds_hist + k_ds_pass x npass: stable LSD radix sort of the visible
//      Gaussians (tiles_touched > 0) by their fp32 depth bits relative to
//      bits(z_near) (visible depths lie in [z_near, z_far], so the keys span
//      nbits(bits(z_far) - bits(z_near)) bits: 27 for 0.2 / 100 m -> 3
//      passes of 9-bit digits).  One histogram kernel for all passes; every
//      pass ranks its 4096-key tile stably per warp (ballot-sliced peer
//      masks), gets its digit offsets from the earlier tiles by decoupled
//      look-back, and scatters.  Positive floats order as their bit patterns
//      and the radix sort is stable on ascending ids: the result is the
//      (depth, id) order.  The last pass also scatters the Gaussians' tile
//      rects into that order.
//   2. k_bin_prefix: the exclusive prefix of the tile counts over that order
//      (decoupled look-back), i.e. the position of every Gaussian's first pair
//      in the flat list F of all pairs in (Gaussian order, rect row-major)
//      order, P = |F|, and for every warp of the next kernels the Gaussian
//      holding its first slot: the pairs, not the Gaussians, are split evenly
//      (near splats have large rects and come first in the order).
//   3. k_bin_count: warp g takes the slots [g C, (g + 1) C) of F (C = 32768 /
//      wb), its CTA counts its pairs per tile (shared-memory counters).
//   4. k_bin_scan: per tile, the exclusive scan of the CTA counts (a warp per
//      tile) and the tile total.
//   5. k_bin_emit: per CTA, the tile starts (scan of the totals), the capacity
//      check, per-warp per-tile offsets (each warp counts its own slots
//      again), then every warp walks its slots in order, 32 per step; slots
//      of one step that hit the same tile come from increasing positions in
//      the order and are ranked by __match_any_sync, so every tile's list
//      receives its Gaussians exactly in (depth, id) order.  CTA 0 also writes
//      the tile ranges, P, the overflow counter and the heaviest-first order.
// Everything is integer arithmetic on the fp32 depth bits: the output is
// bit-deterministic (no atomics decide a position).
#include <algorithm>
#include <cstring>

#include "gs_internal.cuh"

namespace gs {

constexpr int kDsThreads = 512;                 // sort-pass CTA: 16 warps
constexpr int kDsWarps = kDsThreads / 32;
constexpr int kDsItems = 8;                     // keys per thread
constexpr int kDsTile = kDsThreads * kDsItems;  // 4096 keys per sort-pass CTA
constexpr int kDsMaxBits = 11;                  // digit bits per pass (<= 2048 digits)
constexpr int kHistThreads = 256;
constexpr int kBlockPairs = 32768;              // pair slots per count / emit CTA (wb warps)
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1u;

struct BinLayout {
  int n, T, TX, TY;
  int64_t capacity;
  uint32_t kbase, kmax;  // key = depth bits - kbase, in [0, kmax]
  int npass, dbits, ndig;
  int gsort;  // sort-pass CTAs (from n)
  int wb;     // warps per count / emit CTA
  int gbin;   // count / emit CTAs (from the capacity)
  size_t hist, ctr, status, pstatus, misc, zero_end;
  size_t key0, val0, key1, val1, srect, pre, wstart, cnt, totals, total;
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static uint32_t f2u(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

static int host_nbits(uint32_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// warps per count / emit CTA: the emit CTA holds wb x T u16 offsets + T u32 bases
static int bin_warps(int T) {
  for (int wb = 16; wb >= 1; wb >>= 1)
    if (size_t(wb) * T * 2 + size_t(T) * 4 + 1024 <= 200 * 1024) return wb;
  return 0;
}

static bool make_layout(int32_t n, int64_t capacity, const gs_camera &cam, BinLayout &L) {
  L.n = n;
  L.capacity = capacity;
  L.TX = tiles_x(cam);
  L.TY = tiles_y(cam);
  L.T = L.TX * L.TY;
  if (L.T > (1 << 21) || capacity >= (int64_t(1) << 30) || n >= (1 << 30)) return false;
  L.wb = bin_warps(L.T);
  if (L.wb == 0) return false;
  L.kbase = f2u(cam.z_near);
  L.kmax = f2u(cam.z_far) - L.kbase;
  const int nb = std::max(1, host_nbits(L.kmax));
  L.npass = (nb + kDsMaxBits - 1) / kDsMaxBits;
  L.dbits = (nb + L.npass - 1) / L.npass;
  L.ndig = 1 << L.dbits;
  const int nn = n > 0 ? n : 1;
  L.gsort = (nn + kDsTile - 1) / kDsTile;
  const int64_t cap = capacity > 0 ? capacity : 1;
  L.gbin = int((cap + kBlockPairs - 1) / kBlockPairs);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  L.hist = take(size_t(4) * L.npass * L.ndig);
  L.ctr = take(4 * 8);
  L.status = take(size_t(4) * L.npass * L.gsort * L.ndig);
  L.pstatus = take(size_t(4) * L.gsort);  // k_bin_prefix look-back words
  L.misc = take(4 * 8);                   // [0] P
  L.zero_end = off;
  L.key0 = take(size_t(4) * nn);
  L.val0 = take(size_t(4) * nn);
  L.key1 = take(size_t(4) * nn);
  L.val1 = take(size_t(4) * nn);
  L.srect = take(size_t(8) * nn);
  L.pre = take(size_t(4) * nn);
  L.wstart = take(size_t(4) * L.gbin * L.wb);
  L.cnt = take(size_t(4) * L.T * L.gbin);
  L.totals = take(size_t(4) * L.T);
  L.total = off;
  return true;
}

// ---------------------------------------------------------------------------
// warp / block primitives

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Block exclusive scan of one value per thread (blockDim multiple of 32, <= 1024).
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t *sh /* >= 33 */, uint32_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t inc = warp_incl_scan(v);
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t s = lane < nw ? sh[lane] : 0;
    const uint32_t si = warp_incl_scan(s);
    if (lane < nw) sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  const uint32_t r = inc - v + sh[w];
  total = sh[32];
  __syncthreads();
  return r;
}

// In place: a[0..n) <- exclusive prefix sums (block-wide, blockDim threads,
// n / blockDim consecutive entries per thread); returns the total.
__device__ uint32_t block_excl_scan_array(uint32_t *a, int n, uint32_t *sh) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  uint32_t s = 0;
  for (int k = 0; k < per; ++k)
    if (b0 + k < n) s += a[b0 + k];
  uint32_t total;
  uint32_t ex = block_excl_scan(s, sh, total);
  for (int k = 0; k < per; ++k)
    if (b0 + k < n) {
      const uint32_t c = a[b0 + k];
      a[b0 + k] = ex;
      ex += c;
    }
  __syncthreads();
  return total;
}

// Lanes of `act` whose digit equals this lane's: one ballot per digit bit.
// Every lane of the warp must call it.
__device__ __forceinline__ unsigned peer_mask(unsigned act, uint32_t d, int dbits) {
  unsigned m = act;
#pragma unroll
  for (int b = 0; b < kDsMaxBits; ++b) {
    if (b >= dbits) break;
    const bool bit = (d >> b) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bb : ~bb;
  }
  return m;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------
// Stage 1: stable LSD radix sort of the visible Gaussians by depth bits.

struct DsArgs {
  const float *depth;
  const int32_t *tiles_touched;
  const short4 *rect;
  int n;
  uint32_t kbase, kmax;
  int npass, dbits, ndig, gsort;
  uint32_t *hist;    // [npass][ndig] global digit counts
  uint32_t *ctr;     // [npass] virtual CTA counters
  uint32_t *status;  // [npass][gsort][ndig] look-back words
  uint32_t *key[2], *val[2];
  short4 *srect;     // the rects in the final order
};

__device__ __forceinline__ uint32_t depth_key(const DsArgs &a, int i) {
  // visible depths are RN(p_z) with z_near <= p_z <= z_far (gs_project), so
  // the key lies in [0, kmax]; the clamp only guards the digit range
  return min(__float_as_uint(__ldg(a.depth + i)) - a.kbase, a.kmax);
}

__global__ void __launch_bounds__(kHistThreads) k_ds_hist(DsArgs a) {
  pdl_begin();
  extern __shared__ uint32_t s_h[];  // [npass][ndig]
  const int nh = a.npass * a.ndig;
  for (int i = threadIdx.x; i < nh; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const uint32_t mask = uint32_t(a.ndig - 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
    if (__ldg(a.tiles_touched + i) > 0) {
      const uint32_t k = depth_key(a, i);
      for (int p = 0; p < a.npass; ++p) atomicAdd(&s_h[p * a.ndig + ((k >> (p * a.dbits)) & mask)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nh; i += blockDim.x)
    if (s_h[i]) atomicAdd(a.hist + i, s_h[i]);
}

// One stable pass on digit p.  Keys are held "blocked": warp w owns the
// positions [w 32 I, (w + 1) 32 I) of the CTA's tile, its k-th round the 32
// positions w 32 I + 32 k + lane (I = kDsItems).
__global__ void __launch_bounds__(kDsThreads) k_ds_pass(DsArgs a, int p) {
  pdl_begin();
  extern __shared__ uint32_t s_dyn[];
  uint16_t *s_cnt = reinterpret_cast<uint16_t *>(s_dyn);            // [kDsWarps][ndig]: counts -> warp offsets
  uint32_t *s_off = s_dyn + (kDsWarps * a.ndig) / 2;               // [ndig]: global digit base + earlier tiles
  __shared__ uint32_t sh[33];
  __shared__ int s_vb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nd = a.ndig;
  const uint32_t mask = uint32_t(nd - 1);
  const int shift = p * a.dbits;
  if (threadIdx.x == 0) s_vb = int(atomicAdd(a.ctr + p, 1u));  // virtual CTA id: predecessors have started
  // global digit bases of this pass (exclusive scan of its histogram); the
  // visible count = the total of any pass's histogram
  for (int d = threadIdx.x; d < nd; d += blockDim.x) s_off[d] = a.hist[p * nd + d];
  __syncthreads();
  const uint32_t nvis = block_excl_scan_array(s_off, nd, sh);
  const int vb = s_vb;
  const int nin = p == 0 ? a.n : int(nvis);
  if (vb * kDsTile >= nin) return;  // empty tile: no later tile reads its status
  for (int i = threadIdx.x; i < kDsWarps * nd / 2; i += blockDim.x) s_dyn[i] = 0u;
  __syncthreads();
  // load (pass 0: the visible Gaussians of the index range, id = index)
  const uint32_t *kin = a.key[p & 1], *vin = a.val[p & 1];
  uint32_t key[kDsItems], val[kDsItems];
  bool ok[kDsItems];
  const int base = vb * kDsTile + w * 32 * kDsItems;
#pragma unroll
  for (int k = 0; k < kDsItems; ++k) {
    const int i = base + 32 * k + lane;
    if (p == 0) {
      ok[k] = i < a.n && __ldg(a.tiles_touched + i) > 0;
      key[k] = ok[k] ? depth_key(a, i) : 0u;
      val[k] = uint32_t(i);
    } else {
      ok[k] = i < nin;
      key[k] = ok[k] ? kin[i] : 0u;
      val[k] = ok[k] ? vin[i] : 0u;
    }
  }
  // per-warp stable ranks (rounds in order, lanes in order)
  uint16_t rank[kDsItems];
  uint16_t *cw = s_cnt + w * nd;
#pragma unroll
  for (int k = 0; k < kDsItems; ++k) {
    const unsigned act = __ballot_sync(0xffffffffu, ok[k]);
    const uint32_t d = (key[k] >> shift) & mask;
    const unsigned peers = peer_mask(act, d, a.dbits);
    const uint32_t before = ok[k] ? cw[d] : 0u;
    rank[k] = uint16_t(before + __popc(peers & lanemask_lt()));
    __syncwarp();
    if (ok[k] && lane == 31 - __clz(peers)) cw[d] = uint16_t(before + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  // per digit: the tile's count (published for the look-back) and the warp offsets
  uint32_t *st = a.status + (size_t(p) * a.gsort + vb) * nd;
  for (int d = threadIdx.x; d < nd; d += blockDim.x) {
    uint32_t run = 0;
    for (int ww = 0; ww < kDsWarps; ++ww) {
      const uint32_t c = s_cnt[ww * nd + d];
      s_cnt[ww * nd + d] = uint16_t(run);
      run += c;
    }
    if (vb == 0) {
      st_release(st + d, kFlagInc | run);
    } else {
      st_release(st + d, kFlagAgg | run);
      // decoupled look-back over the earlier tiles of this pass
      uint32_t ex = 0;
      for (int j = vb - 1; j >= 0;) {
        const uint32_t s = ld_acquire(a.status + (size_t(p) * a.gsort + j) * nd + d);
        if (!(s & ~kValMask)) continue;  // not published yet: spin
        ex += s & kValMask;
        if (s & kFlagInc) break;
        --j;
      }
      st_release(st + d, kFlagInc | (ex + run));
      s_off[d] += ex;
    }
  }
  __syncthreads();
  // scatter (the last pass also moves the rects into the final order)
  const bool last = p == a.npass - 1;
  uint32_t *kout = a.key[(p + 1) & 1], *vout = a.val[(p + 1) & 1];
#pragma unroll
  for (int k = 0; k < kDsItems; ++k) {
    if (!ok[k]) continue;
    const uint32_t d = (key[k] >> shift) & mask;
    const uint32_t pos = s_off[d] + s_cnt[w * nd + d] + rank[k];
    kout[pos] = key[k];
    vout[pos] = val[k];
    if (last) a.srect[pos] = __ldg(a.rect + val[k]);
  }
}

// ---------------------------------------------------------------------------
// Stages 2-4: stable per-tile emission over the (depth, id) order.

struct BinArgs {
  const uint32_t *hist;   // pass-0 digit counts (their total = visible count)
  int ndig;
  const uint32_t *ids;    // [nvis] Gaussian ids in (depth, id) order
  const short4 *srect;    // [nvis] their rects
  uint32_t *pre;          // [nvis] flat position of each Gaussian's first pair
  uint32_t *wstart;       // [gbin wb] per warp: the Gaussian holding its first slot
  uint32_t *pstatus;      // [gsort] k_bin_prefix look-back words
  uint32_t *ctr;          // virtual CTA counter of k_bin_prefix
  uint32_t *misc;         // [0] P
  int TX, TY, T, gbin, wb;
  uint32_t cw;            // pair slots per warp (kBlockPairs / wb)
  uint32_t *cnt;          // [T][gbin]: CTA counts -> exclusive prefix over CTAs
  uint32_t *totals;       // [T]
  int64_t capacity;
  int32_t *sorted_idx, *tile_range, *tile_order;
  int64_t *n_pairs;
  gs_counters *cntrs;
};

__device__ __forceinline__ uint32_t visible_count(const BinArgs &a, uint32_t *sh) {
  uint32_t s = 0;
  for (int d = threadIdx.x; d < a.ndig; d += blockDim.x) s += a.hist[d];
  uint32_t total;
  block_excl_scan(s, sh, total);
  return total;
}

__device__ __forceinline__ uint32_t rect_area(short4 r) {
  return (r.z >= r.x && r.w >= r.y) ? uint32_t(r.z - r.x + 1) * uint32_t(r.w - r.y + 1) : 0u;
}

// Exclusive prefix of the tile counts over the (depth, id) order: 4096
// Gaussians per CTA (512 threads x 8 consecutive), decoupled look-back on the
// CTA sums; also the first Gaussian of every warp's slot range and P.
__global__ void __launch_bounds__(kDsThreads) k_bin_prefix(BinArgs a) {
  pdl_begin();
  __shared__ uint32_t sh[33];
  __shared__ int s_vb;
  __shared__ uint32_t s_ex;
  const uint32_t nvis = visible_count(a, sh);
  if (threadIdx.x == 0) s_vb = int(atomicAdd(a.ctr, 1u));
  __syncthreads();
  const int vb = s_vb;
  if (vb * kDsTile >= int(nvis)) return;
  const int k0 = vb * kDsTile + threadIdx.x * kDsItems;
  uint32_t c[kDsItems], sum = 0;
#pragma unroll
  for (int k = 0; k < kDsItems; ++k) {
    c[k] = k0 + k < int(nvis) ? rect_area(a.srect[k0 + k]) : 0u;
    sum += c[k];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan(sum, sh, tot);
  if (threadIdx.x == 0) {
    uint32_t e = 0;
    if (vb == 0) {
      st_release(a.pstatus, kFlagInc | tot);
    } else {
      st_release(a.pstatus + vb, kFlagAgg | tot);
      for (int j = vb - 1; j >= 0;) {
        const uint32_t s = ld_acquire(a.pstatus + j);
        if (!(s & ~kValMask)) continue;  // not published yet: spin
        e += s & kValMask;
        if (s & kFlagInc) break;
        --j;
      }
      st_release(a.pstatus + vb, kFlagInc | (e + tot));
    }
    s_ex = e;
    if ((vb + 1) * kDsTile >= int(nvis)) a.misc[0] = e + tot;  // the last CTA: P
  }
  __syncthreads();
  ex += s_ex;
#pragma unroll
  for (int k = 0; k < kDsItems; ++k) {
    if (k0 + k >= int(nvis)) break;
    a.pre[k0 + k] = ex;
    // warp slot ranges starting inside this Gaussian's pairs
    for (uint32_t q = (ex + a.cw - 1) / a.cw * a.cw; q < ex + c[k]; q += a.cw) a.wstart[q / a.cw] = uint32_t(k0 + k);
    ex += c[k];
  }
}

// The pairs of flat slots [q0, q1) of F, warp-wide, 32 per step, starting at
// Gaussian k (the one holding slot q0): f(j, tile, valid, kw) per step, where
// lane j of the current window of 32 Gaussians (kw = its first) holds the
// slot's Gaussian; all lanes call f every step (valid = false past the end).
template <class F>
__device__ __forceinline__ void for_warp_pairs(const BinArgs &a, uint32_t nvis, uint32_t q0, uint32_t q1, int k,
                                               F &&f) {
  const int lane = threadIdx.x & 31;
  for (;; k += 32) {
    const int kk = k + lane;
    const short4 r = kk < int(nvis) ? a.srect[kk] : make_short4(0, 0, -1, -1);
    const uint32_t Q = a.pre[k];
    const int wdt = r.z - r.x + 1;
    const int nt = int(rect_area(r));
    const int incl = int(warp_incl_scan(uint32_t(nt)));
    const uint32_t total = uint32_t(__shfl_sync(0xffffffffu, incl, 31));
    const int xy = (int(r.x) & 0xffff) | (int(r.y) << 16);
    // row = floor(local / wdt) as floor((local + 0.5) (1 / wdt)) in fp32: exact
    // (local < 2^22; the quotient is >= 0.5 / wdt away from an integer)
    const float iw = 1.0f / float(max(wdt, 1));
    const uint32_t pa = q0 > Q ? q0 - Q : 0u, pb = min(q1 - Q, total);
    for (uint32_t p0 = pa; p0 < pb; p0 += 32) {
      const int p = int(p0) + lane;
      // j = number of lanes whose inclusive prefix is <= p
      int j = 0;
#pragma unroll
      for (int b = 16; b > 0; b >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, j + b - 1);
        j += v <= p ? b : 0;
      }
      j = min(j, 31);
      const int ij = __shfl_sync(0xffffffffu, incl, j), nj = __shfl_sync(0xffffffffu, nt, j);
      const int xyj = __shfl_sync(0xffffffffu, xy, j), wj = __shfl_sync(0xffffffffu, wdt, j);
      const float iwj = __shfl_sync(0xffffffffu, iw, j);
      int tile = 0;
      const bool valid = uint32_t(p) < pb;
      if (valid) {
        const int local = p - (ij - nj);
        const int row = int((float(local) + 0.5f) * iwj);
        const int col = local - row * wj;
        tile = ((xyj >> 16) + row) * a.TX + (xyj & 0xffff) + col;
      }
      f(j, tile, valid, k);
    }
    if (Q + total >= q1) break;
  }
}

// P and this warp's slot range [q0, q1) (empty past P)
__device__ __forceinline__ void warp_slots(const BinArgs &a, uint32_t P, uint32_t &q0, uint32_t &q1, int &k) {
  const uint32_t g = blockIdx.x * a.wb + (threadIdx.x >> 5);
  q0 = g * a.cw;
  q1 = min(q0 + a.cw, P);
  k = q0 < P ? int(a.wstart[g]) : 0;
}

__global__ void __launch_bounds__(512) k_bin_count(BinArgs a) {
  pdl_begin();
  extern __shared__ uint32_t s_c[];  // [T]
  __shared__ uint32_t sh[33];
  const uint32_t nvis = visible_count(a, sh);
  const uint32_t P = nvis ? a.misc[0] : 0u;
  if (uint64_t(blockIdx.x) * kBlockPairs >= P) return;  // k_bin_scan reads only the CTAs holding pairs
  for (int t = threadIdx.x; t < a.T; t += blockDim.x) s_c[t] = 0;
  __syncthreads();
  uint32_t q0, q1;
  int k;
  warp_slots(a, P, q0, q1, k);
  if (q0 < q1)
    for_warp_pairs(a, nvis, q0, q1, k, [&](int, int tile, bool valid, int) {
      if (valid) atomicAdd(&s_c[tile], 1u);
    });
  __syncthreads();
  for (int t = threadIdx.x; t < a.T; t += blockDim.x) a.cnt[size_t(t) * a.gbin + blockIdx.x] = s_c[t];
}

// one warp per tile: exclusive scan of its CTA counts, the tile total
__global__ void __launch_bounds__(256) k_bin_scan(BinArgs a) {
  pdl_begin();
  __shared__ uint32_t sh[33];
  const int lane = threadIdx.x & 31;
  const uint32_t nvis = visible_count(a, sh);
  const uint32_t P = nvis ? a.misc[0] : 0u;
  const int nb = min(int((uint64_t(P) + kBlockPairs - 1) / kBlockPairs), a.gbin);
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= a.T) return;
  uint32_t *c = a.cnt + size_t(t) * a.gbin;
  uint32_t carry = 0;
  for (int b0 = 0; b0 < nb; b0 += 32) {
    const int b = b0 + lane;
    const uint32_t v = b < nb ? c[b] : 0u;
    const uint32_t inc = warp_incl_scan(v) + carry;
    if (b < nb) c[b] = inc - v;
    carry = __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) a.totals[t] = carry;
}

__global__ void __launch_bounds__(512) k_bin_emit(BinArgs a) {
  pdl_begin();
  extern __shared__ uint32_t s_e[];  // [T] tile bases, then [wb][T] u16 per-warp offsets
  __shared__ uint32_t sh[33];
  __shared__ unsigned s_b[64];
  __shared__ uint32_t s_max;
  const int wb = a.wb, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int T = a.T;
  uint32_t *s_base = s_e;
  uint16_t *s_off = reinterpret_cast<uint16_t *>(s_e + T);
  const uint32_t nvis = visible_count(a, sh);
  const uint32_t P = nvis ? a.misc[0] : 0u;
  const bool over = int64_t(P) > a.capacity;
  const bool has = !over && uint64_t(blockIdx.x) * kBlockPairs < P;
  if (!has && blockIdx.x != 0) return;
  // the tile totals (no pair: never computed; overflow: the lists stay empty)
  auto total_of = [&](int t) { return (over || P == 0) ? 0u : a.totals[t]; };
  // tile starts: exclusive scan of the totals
  for (int t = threadIdx.x; t < T; t += blockDim.x) s_base[t] = total_of(t);
  __syncthreads();
  block_excl_scan_array(s_base, T, sh);
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
      const int st = int(s_base[t]);
      reinterpret_cast<int2 *>(a.tile_range)[t] = make_int2(st, st + int(total_of(t)));
    }
    if (threadIdx.x == 0) {
      *a.n_pairs = int64_t(P);
      if (over && a.cntrs) atomicAdd(reinterpret_cast<unsigned long long *>(&a.cntrs->n_overflow), 1ull);
    }
  }
  if (has) {
    // this CTA's base per tile, per-warp counts (each warp its own row)
    for (int t = threadIdx.x; t < T; t += blockDim.x) s_base[t] += a.cnt[size_t(t) * a.gbin + blockIdx.x];
    for (int i = threadIdx.x; i < (wb * T + 1) / 2; i += blockDim.x) reinterpret_cast<uint32_t *>(s_off)[i] = 0u;
    __syncthreads();
    uint16_t *row = s_off + w * T;
    uint32_t q0, q1;
    int k;
    warp_slots(a, P, q0, q1, k);
    if (q0 < q1)
      for_warp_pairs(a, nvis, q0, q1, k, [&](int, int tile, bool valid, int) {
        // lanes of one step that hit the same tile form a match group
        const unsigned g = __match_any_sync(0xffffffffu, valid ? tile : -1);
        if (valid && lane == __ffs(g) - 1) row[tile] = uint16_t(row[tile] + __popc(g));
        __syncwarp();
      });
    __syncthreads();
    // per tile: exclusive prefix over the warps
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
      uint32_t run = 0;
      for (int ww = 0; ww < wb; ++ww) {
        const uint32_t c = s_off[ww * T + t];
        s_off[ww * T + t] = uint16_t(run);
        run += c;
      }
    }
    __syncthreads();
    // emission in order: position = tile base + warp offset + pairs of this
    // tile earlier in the warp's walk (earlier steps: the running offset;
    // this step: lanes below in the match group, which hold earlier Gaussians)
    if (q0 < q1) {
      int kw = -1, id = 0;
      for_warp_pairs(a, nvis, q0, q1, k, [&](int j, int tile, bool valid, int kwin) {
        if (kwin != kw) {  // a new window of 32 Gaussians: their ids
          kw = kwin;
          id = kw + lane < int(nvis) ? int(a.ids[kw + lane]) : 0;
        }
        const int gid = __shfl_sync(0xffffffffu, id, j);
        const unsigned g = __match_any_sync(0xffffffffu, valid ? tile : -1);
        if (valid) a.sorted_idx[s_base[tile] + row[tile] + __popc(g & lanemask_lt())] = gid;
        __syncwarp();
        if (valid && lane == __ffs(g) - 1) row[tile] = uint16_t(row[tile] + __popc(g));
        __syncwarp();
      });
    }
  }
  if (blockIdx.x != 0 || !a.tile_order) return;
  // CTA 0: tiles by descending list length, 64 buckets of max/64 (order
  // inside a bucket unspecified), a scheduling hint for the compositing
  __syncthreads();
  if (threadIdx.x == 0) s_max = 0;
  if (threadIdx.x < 64) s_b[threadIdx.x] = 0;
  __syncthreads();
  uint32_t m = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) m = max(m, total_of(t));
  atomicMax(&s_max, m);
  __syncthreads();
  const int64_t den = int64_t(s_max) + 1;
  for (int t = threadIdx.x; t < T; t += blockDim.x)
    atomicAdd(&s_b[63 - int(int64_t(total_of(t)) * 64 / den)], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int b = 0; b < 64; ++b) {
      const unsigned c = s_b[b];
      s_b[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x)
    a.tile_order[atomicAdd(&s_b[63 - int(int64_t(total_of(t)) * 64 / den)], 1u)] = t;
}

// Tiles by descending work, 64 buckets of max/64 (single CTA).
__global__ void __launch_bounds__(1024) k_order_by_work(const int32_t *__restrict__ work, int T, int32_t *order) {
  // no early trigger: a backward launched after this kernel with tile_done
  // does not wait for its predecessor grid, and it reads this order
  pdl_wait();
  __shared__ int s_max;
  __shared__ unsigned s_b[64];
  if (threadIdx.x == 0) s_max = 0;
  if (threadIdx.x < 64) s_b[threadIdx.x] = 0;
  __syncthreads();
  int m = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) m = max(m, work[t]);
  atomicMax(&s_max, m);
  __syncthreads();
  const int64_t den = int64_t(s_max) + 1;
  for (int t = threadIdx.x; t < T; t += blockDim.x)
    atomicAdd(&s_b[63 - int(int64_t(max(work[t], 0)) * 64 / den)], 1u);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int b = 0; b < 64; ++b) {
      const unsigned c = s_b[b];
      s_b[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x)
    order[atomicAdd(&s_b[63 - int(int64_t(max(work[t], 0)) * 64 / den)], 1u)] = t;
}

}  // namespace gs

extern "C" int gs_tile_order(const int32_t *work, int32_t T, int32_t *order, void *stream) {
  using namespace gs;
  if (!work || !order || T <= 0) {
    set_error("gs_tile_order: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  launch_pdl(k_order_by_work, dim3(1), dim3(1024), 0, as_stream(stream), work, T, order);
  return check_launch("gs_tile_order");
}

extern "C" size_t gs_binsort_workspace_bytes(int32_t n, int64_t capacity, gs_camera cam) {
  gs::BinLayout L;
  if (n < 0 || capacity < 0 || !gs::camera_ok(cam) || !gs::make_layout(n, capacity, cam, L)) return 0;
  return L.total;
}

extern "C" int gs_bin_sort(gs_proj pr, int32_t n, gs_camera cam, void *ws, size_t ws_bytes, int64_t capacity,
                           int32_t *sorted_idx, int32_t *tile_range, int32_t *tile_order, int64_t *n_pairs,
                           gs_counters *cnt, void *stream) {
  using namespace gs;
  if (n < 0 || !camera_ok(cam) || !tile_range || !n_pairs || capacity < 0 || (capacity > 0 && !sorted_idx)) {
    set_error("gs_bin_sort: invalid argument");
    return GS_ERR_INVALID_ARG;
  }
  if (n > 0 && (!pr.depth || !pr.rect || !pr.tiles_touched || (reinterpret_cast<uintptr_t>(pr.rect) & 7u))) {
    set_error("gs_bin_sort: null or misaligned projection arrays");
    return GS_ERR_INVALID_ARG;
  }
  BinLayout L;
  if (!make_layout(n, capacity, cam, L)) {
    set_error("gs_bin_sort: problem too large (n=%d, capacity=%lld, tiles=%d)", n, (long long)capacity,
              tiles_x(cam) * tiles_y(cam));
    return GS_ERR_UNSUPPORTED;
  }
  if (!ws || ws_bytes < L.total || (reinterpret_cast<uintptr_t>(ws) & 15u)) {
    set_error("gs_bin_sort: workspace %zu < %zu bytes (or misaligned)", ws_bytes, L.total);
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char *w = static_cast<char *>(ws);
  auto U = [&](size_t off) { return reinterpret_cast<uint32_t *>(w + off); };
  cudaMemsetAsync(w, 0, L.zero_end, s);
  DsArgs d{pr.depth, pr.tiles_touched, reinterpret_cast<const short4 *>(pr.rect), n, L.kbase, L.kmax, L.npass,
           L.dbits, L.ndig, L.gsort, U(L.hist), U(L.ctr), U(L.status), {U(L.key0), U(L.key1)},
           {U(L.val0), U(L.val1)}, reinterpret_cast<short4 *>(w + L.srect)};
  const uint32_t *ids = (L.npass & 1) ? U(L.val1) : U(L.val0);  // pass p writes val[(p + 1) & 1]
  const size_t ds_smem = size_t(kDsWarps) * L.ndig * 2 + size_t(L.ndig) * 4;
  const size_t cnt_smem = size_t(L.T) * 4;
  const size_t emit_smem = size_t(L.T) * 4 + ((size_t(L.wb) * L.T * 2 + 3) & ~size_t(3));
  static thread_local size_t smem_set = 0;
  const size_t need = std::max(std::max(ds_smem, emit_smem), cnt_smem);
  if (need > 48 * 1024 && need > smem_set) {
    cudaFuncSetAttribute(k_ds_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max(ds_smem, size_t(48) << 10)));
    cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max(cnt_smem, size_t(48) << 10)));
    cudaFuncSetAttribute(k_bin_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max(emit_smem, size_t(48) << 10)));
    smem_set = need;
  }
  BinArgs b{U(L.hist), L.ndig, ids, reinterpret_cast<const short4 *>(w + L.srect), U(L.pre), U(L.wstart),
            U(L.pstatus), U(L.ctr) + 4, U(L.misc), L.TX, L.TY, L.T, L.gbin, L.wb, uint32_t(kBlockPairs / L.wb),
            U(L.cnt), U(L.totals), capacity, sorted_idx, tile_range, tile_order, n_pairs, cnt};
  if (n > 0) {
    const int hb = std::max(1, std::min(2 * 148, (n + 4 * kHistThreads - 1) / (4 * kHistThreads)));
    launch_pdl(k_ds_hist, dim3(hb), dim3(kHistThreads), size_t(4) * L.npass * L.ndig, s, d);
    for (int p = 0; p < L.npass; ++p) launch_pdl(k_ds_pass, dim3(L.gsort), dim3(kDsThreads), ds_smem, s, d, p);
    launch_pdl(k_bin_prefix, dim3(L.gsort), dim3(kDsThreads), 0, s, b);
    launch_pdl(k_bin_count, dim3(L.gbin), dim3(32 * L.wb), cnt_smem, s, b);
    launch_pdl(k_bin_scan, dim3((L.T + 7) / 8), dim3(256), 0, s, b);
  }
  launch_pdl(k_bin_emit, dim3(L.gbin), dim3(32 * L.wb), emit_smem, s, b);
  return check_launch("gs_bin_sort");
}
