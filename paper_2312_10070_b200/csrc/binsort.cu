// binsort.cu — S2 gs_bin_sort: tile binning with deterministic depth order
// ("m ordered Gaussians"; R10).
//
// Result = every (tile, Gaussian) pair ordered by the composite key
// (tile asc, fp32 depth asc, Gaussian id asc), computed in two stable stages
// that together equal one LSD radix sort on that key while moving ~4x fewer
// bytes than sorting 64-bit pair keys:
//   1. stable LSD radix sort of the VISIBLE Gaussians by depth bits
//      (9-bit digits; the visibility filter is fused into pass 0, whose input
//      order is the Gaussian id, so equal depths stay in id order);
//   2. one stable counting sort of the pair stream (depth-sorted Gaussians x
//      their rect tiles, row-major) by tile id: per-block tile histograms,
//      a device-wide exclusive scan in tile-major order, then a scatter in
//      which each warp walks its pairs 32 at a time and ranks equal tiles
//      with __match_any_sync, so ties keep stream order.
// Every counter is an integer: the output is bit-deterministic.
#include <algorithm>
#include <cstring>

#include "gs_internal.cuh"

namespace gs {

constexpr int kRBits = 9;
constexpr int kRDigits = 1 << kRBits;
constexpr int kRThreads = 256;
constexpr int kRItems = 8;
constexpr int kRTile = kRThreads * kRItems;  // 2048 keys per radix block
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096
constexpr int kScanMaxBlocks = 4096;                  // one 1024x4 block scans the sums
constexpr int kMaxBinSmem = 227 * 1024;

struct SortLayout {
  int n, T, TX, tbits;
  int passes;
  uint32_t zbase;
  int nblk_r;   // radix blocks
  int nblk_b;   // bin blocks
  int W;        // warps per bin block
  int nchunks;  // nblk_b * W pair-balanced chunks, one per warp
  size_t keys_a, keys_b, vals_a, vals_b, rhist, thist, cstart, sums, misc, total;
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static bool make_layout(int32_t n, const gs_camera &cam, SortLayout &L) {
  L.n = n;
  L.TX = tiles_x(cam);
  L.T = L.TX * tiles_y(cam);
  L.tbits = 1;
  while ((1 << L.tbits) < L.T) ++L.tbits;
  // significant bits of (bits(z_far) - bits(z_near)): positive floats order as uints
  uint32_t zb, ze;
  float zn = cam.z_near, zf = cam.z_far;
  memcpy(&zb, &zn, 4);
  memcpy(&ze, &zf, 4);
  L.zbase = zb;
  uint32_t range = ze - zb;
  int bits = range ? 32 - __builtin_clz(range) : 1;
  L.passes = (bits + kRBits - 1) / kRBits;
  L.nblk_r = (n + kRTile - 1) / kRTile;
  if (L.nblk_r < 1) L.nblk_r = 1;
  // bin blocks: W warps, smem = 4T (block base) + 2 W T (per-warp u16 counts)
  L.W = 8;
  while (L.W > 1 && size_t(4 + 2 * L.W) * L.T > size_t(kMaxBinSmem)) L.W >>= 1;
  if (size_t(4 + 2 * L.W) * L.T > size_t(kMaxBinSmem)) return false;
  L.nblk_b = std::min(296, std::max(1, n / 1024));  // 2 x 148 SMs for large problems
  L.nchunks = L.nblk_b * L.W;
  if ((int64_t)L.T * L.nblk_b > (int64_t)kScanTile * kScanMaxBlocks) return false;
  if ((int64_t)kRDigits * L.nblk_r > (int64_t)kScanTile * kScanMaxBlocks) return false;
  if ((int64_t)n > (int64_t)kScanTile * kScanMaxBlocks) return false;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  size_t nn = size_t(n > 0 ? n : 1);
  L.keys_a = take(4 * nn);
  L.keys_b = take(4 * nn);
  L.vals_a = take(4 * nn);
  L.vals_b = take(4 * nn);
  L.rhist = take(4 * size_t(kRDigits) * L.nblk_r);
  L.thist = take(4 * size_t(L.T) * L.nblk_b);
  L.cstart = take(4 * size_t(L.nchunks + 1));
  L.sums = take(4 * size_t(kScanMaxBlocks + 1));
  L.misc = take(64);
  L.total = off;
  return true;
}

// Lanes of `act` whose key agrees with this lane's in its low `bits` bits:
// one ballot per bit (bit-sliced equality).  Every lane of the warp must call
// it; MATCH.ANY is avoided because its latency grows with the number of
// distinct keys in the warp (measured: 1.1 ms for the tile scatter).
template <int kBits>
__device__ __forceinline__ unsigned peer_mask(unsigned act, uint32_t key) {
  unsigned m = act;
#pragma unroll
  for (int b = 0; b < kBits; ++b) {
    const bool bit = (key >> b) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bb : ~bb;
  }
  return m;
}

__device__ __forceinline__ unsigned peer_mask_rt(unsigned act, uint32_t key, int bits) {
  unsigned m = act;
  for (int b = 0; b < bits; ++b) {
    const bool bit = (key >> b) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bb : ~bb;
  }
  return m;
}

// ---------------------------------------------------------------------------
// Device-wide exclusive scan of uint32 counts (in place) + total.

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Block exclusive scan of one value per thread (blockDim multiple of 32, <= 1024).
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t *sh /* >= 33 */, uint32_t &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t inc = warp_incl_scan(v);
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < nw ? sh[lane] : 0;
    uint32_t si = warp_incl_scan(s);
    if (lane < nw) sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  uint32_t r = inc - v + sh[w];
  total = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t *a, int64_t L, const uint32_t *dlen,
                                                               uint32_t *sums) {
  __shared__ uint32_t sh[33];
  if (dlen) L = min(L, int64_t(*dlen));
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + int64_t(k) * kScanThreads + threadIdx.x;
    if (i < L) s += a[i];
  }
  uint32_t tot;
  block_excl_scan(s, sh, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_sums(uint32_t *sums, int nb, uint32_t *total_out) {
  __shared__ uint32_t sh[33];
  uint32_t v[4];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int i = threadIdx.x * 4 + k;
    v[k] = i < nb ? sums[i] : 0;
    s += v[k];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan(s, sh, tot);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int i = threadIdx.x * 4 + k;
    if (i < nb) sums[i] = ex;
    ex += v[k];
  }
  if (threadIdx.x == 0 && total_out) *total_out = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(uint32_t *a, int64_t L, const uint32_t *dlen,
                                                              const uint32_t *sums) {
  __shared__ uint32_t sh[33];
  if (dlen) L = min(L, int64_t(*dlen));
  const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    v[k] = i < L ? a[i] : 0;
    s += v[k];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan(s, sh, tot) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = base + k;
    if (i < L) a[i] = ex;
    ex += v[k];
  }
}

// Exclusive scan of a[0, min(L, *dlen)) (dlen: optional device length).
static void scan_exclusive(uint32_t *a, int64_t L, uint32_t *sums, uint32_t *total, cudaStream_t s,
                           const uint32_t *dlen = nullptr) {
  int nb = int((L + kScanTile - 1) / kScanTile);
  if (nb < 1) nb = 1;
  k_scan_reduce<<<nb, kScanThreads, 0, s>>>(a, L, dlen, sums);
  k_scan_sums<<<1, 1024, 0, s>>>(sums, nb, total);
  k_scan_apply<<<nb, kScanThreads, 0, s>>>(a, L, dlen, sums);
}

// ---------------------------------------------------------------------------
// Stage 1: stable LSD radix sort of visible Gaussians by depth bits.

struct RadixIn {
  // pass 0 reads (depth, tiles_touched) of all n Gaussians; later passes the
  // previous pass's (keys, vals) of length *nvis.
  const float *depth;
  const int32_t *tiles_touched;
  const uint32_t *keys;
  const int32_t *vals;
  const uint32_t *nvis;
  int n;
  uint32_t zbase;
};

__device__ __forceinline__ bool radix_item(const RadixIn &in, bool first, int64_t i, int limit,
                                           uint32_t &key, int32_t &val) {
  key = 0;
  val = 0;
  if (i >= limit) return false;
  if (first) {
    if (__ldg(in.tiles_touched + i) <= 0) return false;
    key = __float_as_uint(__ldg(in.depth + i)) - in.zbase;
    val = int32_t(i);
  } else {
    key = in.keys[i];
    val = in.vals[i];
  }
  return true;
}

__global__ void __launch_bounds__(kRThreads) k_radix_upsweep(RadixIn in, bool first, int shift, int nblk,
                                                             uint32_t *rhist) {
  __shared__ uint32_t h[kRDigits];
  for (int d = threadIdx.x; d < kRDigits; d += kRThreads) h[d] = 0;
  __syncthreads();
  const int limit = first ? in.n : int(*in.nvis);
  const int64_t base = int64_t(blockIdx.x) * kRTile;
#pragma unroll
  for (int k = 0; k < kRItems; ++k) {
    uint32_t key;
    int32_t val;
    if (radix_item(in, first, base + k * kRThreads + threadIdx.x, limit, key, val))
      atomicAdd(&h[(key >> shift) & (kRDigits - 1)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRDigits; d += kRThreads) rhist[size_t(d) * nblk + blockIdx.x] = h[d];
}

// Stable scatter: warp w owns items [base + 256 w, base + 256 (w+1)), walked
// in 8 rounds of 32; ties within a round are ranked by lane (= input order).
// The last pass writes the item's tile count instead of its key: the tile
// counts of the depth-sorted stream, scanned next into pair offsets.
__global__ void __launch_bounds__(kRThreads) k_radix_downsweep(RadixIn in, bool first, bool last, int shift, int nblk,
                                                               const uint32_t *rhist, uint32_t *keys_out,
                                                               int32_t *vals_out) {
  constexpr int kW = kRThreads / 32;
  __shared__ uint32_t wc[kW][kRDigits];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kRDigits; d += kRThreads)
#pragma unroll
    for (int ww = 0; ww < kW; ++ww) wc[ww][d] = 0;
  __syncthreads();
  const int limit = first ? in.n : int(*in.nvis);
  const int64_t base = int64_t(blockIdx.x) * kRTile + int64_t(w) * (32 * kRItems);
  uint32_t key[kRItems];
  int32_t val[kRItems];
  bool ok[kRItems];
#pragma unroll
  for (int r = 0; r < kRItems; ++r) ok[r] = radix_item(in, first, base + r * 32 + lane, limit, key[r], val[r]);
  // walk 1: per-warp digit counts
#pragma unroll 1
  for (int r = 0; r < kRItems; ++r) {
    const unsigned act = __ballot_sync(0xffffffffu, ok[r]);
    const uint32_t d = (key[r] >> shift) & (kRDigits - 1);
    const unsigned peers = peer_mask<kRBits>(act, d);
    if (ok[r] && lane == 31 - __clz(peers)) wc[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive offsets per (warp, digit): global digit offset of this block + earlier warps
  for (int d = threadIdx.x; d < kRDigits; d += kRThreads) {
    uint32_t run = rhist[size_t(d) * nblk + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < kW; ++ww) {
      uint32_t c = wc[ww][d];
      wc[ww][d] = run;
      run += c;
    }
  }
  __syncthreads();
  // walk 2: scatter
#pragma unroll
  for (int r = 0; r < kRItems; ++r) {
    const unsigned act = __ballot_sync(0xffffffffu, ok[r]);
    const uint32_t d = (key[r] >> shift) & (kRDigits - 1);
    const unsigned peers = peer_mask<kRBits>(act, d);
    if (ok[r]) {
      const uint32_t pos = wc[w][d] + __popc(peers & lanemask_lt());
      keys_out[pos] = last ? uint32_t(__ldg(in.tiles_touched + val[r])) : key[r];
      vals_out[pos] = val[r];
    }
    __syncwarp();
    if (ok[r] && lane == 31 - __clz(peers)) wc[w][d] += __popc(peers);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Stage 2: stable counting sort of the pair stream by tile.
//
// poff[r] = exclusive prefix of the tile counts of the depth-sorted stream;
// P = total.  The stream is cut into nchunks pair-balanced chunks of
// Qw = ceil(P / nchunks) pairs (an item belongs to the chunk holding its first
// pair), one chunk per warp, W warps per block: near (large) splats no longer
// pile up in the first blocks.

__global__ void k_chunk_starts(const uint32_t *__restrict__ poff, const uint32_t *__restrict__ nvis,
                               const uint32_t *__restrict__ ptotal, int nchunks, int n, uint32_t *cstart) {
  const int nv = int(*nvis);
  const uint32_t P = *ptotal;
  const uint32_t Qw = max(1u, (P + uint32_t(nchunks) - 1) / uint32_t(nchunks));
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid < nv) {
    const int c = int(poff[gid] / Qw);
    const int cp = gid > 0 ? int(poff[gid - 1] / Qw) : -1;
    for (int k = cp + 1; k <= c && k < nchunks; ++k) cstart[k] = uint32_t(gid);
  }
  if (gid <= nchunks) {
    const int clast = nv > 0 ? int(poff[nv - 1] / Qw) : -1;
    if (gid > clast) cstart[gid] = uint32_t(nv);
  }
}

// One warp walks items [kbeg, kend) of the depth-sorted stream in stream
// order, ONE item per step: lane l takes the item's l-th tile (row-major in its
// rect; items with more than 32 tiles take several steps).  The tiles of one
// item are distinct, so no two lanes of a step touch the same counter and the
// per-tile order is the stream order without any ranking.  Tile (row, col) of
// lane l comes from one multiply-high by ceil(2^32 / width) (exact for
// l, width < 2^16).  wcnt is this warp's u16 tile counter row.
// SCATTER=false counts, SCATTER=true writes sorted_idx.
template <bool SCATTER>
__device__ __forceinline__ void bin_walk(const int32_t *__restrict__ sorted_vals, const short4 *__restrict__ rect,
                                         int kbeg, int kend, int TX, uint16_t *wcnt, const uint32_t *base,
                                         int32_t *sorted_idx) {
  const int lane = threadIdx.x & 31;
  for (int k0 = kbeg; k0 < kend; k0 += 32) {
    // each lane preloads one item of the group
    const int k = k0 + lane;
    int g = 0, rxy = 0, wdt = 1, nt = 0;
    uint32_t magic = 0;
    if (k < kend) {
      g = __ldg(sorted_vals + k);
      const short4 r = __ldg(rect + g);
      wdt = r.z - r.x + 1;
      nt = wdt * (r.w - r.y + 1);
      rxy = (int(r.x) & 0xffff) | (int(r.y) << 16);
      magic = wdt > 1 ? uint32_t((0x100000000ull + uint64_t(wdt) - 1) / uint64_t(wdt)) : 0u;
    }
    const int cnt = min(32, kend - k0);
    for (int i = 0; i < cnt; ++i) {
      const int ig = __shfl_sync(0xffffffffu, g, i);
      const int ixy = __shfl_sync(0xffffffffu, rxy, i);
      const int iw = __shfl_sync(0xffffffffu, wdt, i);
      const int int_ = __shfl_sync(0xffffffffu, nt, i);
      const uint32_t im = __shfl_sync(0xffffffffu, magic, i);
      const int x0 = int(short(ixy & 0xffff)), y0 = ixy >> 16;
      for (int l = lane; l < int_; l += 32) {
        const int row = iw == 1 ? l : int(__umulhi(uint32_t(l), im));
        const int t = (y0 + row) * TX + x0 + (l - row * iw);
        const uint16_t c = wcnt[t];
        if (SCATTER) sorted_idx[base[t] + c] = ig;
        wcnt[t] = uint16_t(c + 1);
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void warp_chunk(const uint32_t *__restrict__ cstart, int W, int &kbeg, int &kend) {
  const int c = blockIdx.x * W + (threadIdx.x >> 5);
  kbeg = int(cstart[c]);
  kend = int(cstart[c + 1]);
}

__global__ void k_bin_count(const int32_t *__restrict__ sorted_vals, const uint32_t *__restrict__ cstart,
                            const short4 *__restrict__ rect, int T, int TX, int tbits, int nblk, uint32_t *thist) {
  extern __shared__ uint32_t smem[];
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5;
  uint16_t *wc = reinterpret_cast<uint16_t *>(smem);
  for (int i = threadIdx.x; i < W * T; i += blockDim.x) wc[i] = 0;
  __syncthreads();
  int kbeg, kend;
  warp_chunk(cstart, W, kbeg, kend);
  bin_walk<false>(sorted_vals, rect, kbeg, kend, TX, wc + size_t(w) * T, nullptr, nullptr);
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    uint32_t c = 0;
    for (int ww = 0; ww < W; ++ww) c += wc[size_t(ww) * T + t];
    thist[size_t(t) * nblk + blockIdx.x] = c;
  }
}

__global__ void k_bin_finish(const uint32_t *thist, int T, int nblk, const uint32_t *ptotal, int64_t capacity,
                             int32_t *tile_range, int64_t *n_pairs, uint32_t *overflow_flag, gs_counters *cnt) {
  const int64_t P = *ptotal;
  const bool over = P > capacity;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    int2 r = make_int2(0, 0);
    if (!over) {
      r.x = int(thist[size_t(t) * nblk]);
      r.y = t + 1 < T ? int(thist[size_t(t + 1) * nblk]) : int(P);
    }
    reinterpret_cast<int2 *>(tile_range)[t] = r;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *n_pairs = P;
    *overflow_flag = over ? 1u : 0u;
    if (over && cnt) atomicAdd(reinterpret_cast<unsigned long long *>(&cnt->n_overflow), 1ull);
  }
}

// Tiles by descending list length, bucketed into 64 classes of
// maxlen/64 (single CTA; order inside a bucket follows the atomics).
__global__ void __launch_bounds__(1024) k_tile_order(const int2 *__restrict__ tile_range, int T, int32_t *order) {
  __shared__ int s_max;
  __shared__ unsigned s_cnt[64];
  if (threadIdx.x == 0) s_max = 0;
  if (threadIdx.x < 64) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  int m = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int2 r = tile_range[t];
    m = max(m, r.y - r.x);
  }
  atomicMax(&s_max, m);
  __syncthreads();
  const int den = s_max + 1;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int2 r = tile_range[t];
    atomicAdd(&s_cnt[63 - int((int64_t(r.y - r.x) * 64) / den)], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int b = 0; b < 64; ++b) {
      const unsigned c = s_cnt[b];
      s_cnt[b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int2 r = tile_range[t];
    order[atomicAdd(&s_cnt[63 - int((int64_t(r.y - r.x) * 64) / den)], 1u)] = t;
  }
}

__global__ void k_bin_scatter(const int32_t *__restrict__ sorted_vals, const uint32_t *__restrict__ cstart,
                              const short4 *__restrict__ rect, int T, int TX, int tbits, int nblk,
                              const uint32_t *__restrict__ thist, const uint32_t *__restrict__ overflow_flag,
                              int32_t *sorted_idx) {
  if (*overflow_flag) return;
  extern __shared__ uint32_t smem[];
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5;
  uint32_t *base = smem;
  uint16_t *wc = reinterpret_cast<uint16_t *>(smem + T);
  for (int i = threadIdx.x; i < W * T; i += blockDim.x) wc[i] = 0;
  __syncthreads();
  int kbeg, kend;
  warp_chunk(cstart, W, kbeg, kend);
  bin_walk<false>(sorted_vals, rect, kbeg, kend, TX, wc + size_t(w) * T, nullptr, nullptr);
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    base[t] = thist[size_t(t) * nblk + blockIdx.x];
    uint32_t run = 0;
    for (int ww = 0; ww < W; ++ww) {
      const uint32_t c = wc[size_t(ww) * T + t];
      wc[size_t(ww) * T + t] = uint16_t(run);
      run += c;
    }
  }
  __syncthreads();
  bin_walk<true>(sorted_vals, rect, kbeg, kend, TX, wc + size_t(w) * T, base, sorted_idx);
}

}  // namespace gs

extern "C" size_t gs_binsort_workspace_bytes(int32_t n, gs_camera cam) {
  gs::SortLayout L;
  if (n < 0 || !gs::camera_ok(cam) || !gs::make_layout(n, cam, L)) return 0;
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
  SortLayout L;
  if (!make_layout(n, cam, L)) {
    set_error("gs_bin_sort: problem too large (n=%d, tiles=%d)", n, tiles_x(cam) * tiles_y(cam));
    return GS_ERR_UNSUPPORTED;
  }
  if (!ws || ws_bytes < L.total) {
    set_error("gs_bin_sort: workspace %zu < %zu bytes", ws_bytes, L.total);
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char *w = static_cast<char *>(ws);
  uint32_t *keys[2] = {reinterpret_cast<uint32_t *>(w + L.keys_a), reinterpret_cast<uint32_t *>(w + L.keys_b)};
  int32_t *vals[2] = {reinterpret_cast<int32_t *>(w + L.vals_a), reinterpret_cast<int32_t *>(w + L.vals_b)};
  uint32_t *rhist = reinterpret_cast<uint32_t *>(w + L.rhist);
  uint32_t *thist = reinterpret_cast<uint32_t *>(w + L.thist);
  uint32_t *cstart = reinterpret_cast<uint32_t *>(w + L.cstart);
  uint32_t *sums = reinterpret_cast<uint32_t *>(w + L.sums);
  uint32_t *misc = reinterpret_cast<uint32_t *>(w + L.misc);  // [0] nvis, [1] P, [2] overflow
  // ---- stage 1: radix passes (pass 0 fuses the visibility filter) ----
  RadixIn in{pr.depth, pr.tiles_touched, nullptr, nullptr, misc + 0, n, L.zbase};
  int cur = 0;
  for (int pass = 0; pass < L.passes; ++pass) {
    const bool first = pass == 0, last = pass == L.passes - 1;
    const int shift = pass * kRBits;
    if (!first) {
      in.keys = keys[cur];
      in.vals = vals[cur];
    }
    const int nxt = first ? 0 : cur ^ 1;
    k_radix_upsweep<<<L.nblk_r, kRThreads, 0, s>>>(in, first, shift, L.nblk_r, rhist);
    scan_exclusive(rhist, int64_t(kRDigits) * L.nblk_r, sums, first ? misc + 0 : nullptr, s);
    k_radix_downsweep<<<L.nblk_r, kRThreads, 0, s>>>(in, first, last, shift, L.nblk_r, rhist, keys[nxt], vals[nxt]);
    cur = nxt;
  }
  const int32_t *svals = vals[cur];
  uint32_t *poff = keys[cur];  // tile counts of the sorted stream -> pair offsets
  // ---- stage 2: tile bucketing ----
  scan_exclusive(poff, int64_t(n > 0 ? n : 1), sums, misc + 1, s, misc + 0);
  {
    const int threads = 256, items = std::max(n, L.nchunks + 1);
    k_chunk_starts<<<(items + threads - 1) / threads, threads, 0, s>>>(poff, misc + 0, misc + 1, L.nchunks, n,
                                                                       cstart);
  }
  const short4 *rect = reinterpret_cast<const short4 *>(pr.rect);
  const size_t count_smem = size_t(2) * L.W * L.T;
  const size_t scat_smem = size_t(4) * L.T + count_smem;
  static thread_local size_t smem_set = 0;
  if (scat_smem > 48 * 1024 && scat_smem > smem_set) {
    cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize, int(scat_smem));
    cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(scat_smem));
    smem_set = scat_smem;
  }
  k_bin_count<<<L.nblk_b, 32 * L.W, count_smem, s>>>(svals, cstart, rect, L.T, L.TX, L.tbits, L.nblk_b, thist);
  scan_exclusive(thist, int64_t(L.T) * L.nblk_b, sums, nullptr, s);
  k_bin_finish<<<(L.T + 255) / 256, 256, 0, s>>>(thist, L.T, L.nblk_b, misc + 1, capacity, tile_range, n_pairs,
                                                  misc + 2, cnt);
  k_bin_scatter<<<L.nblk_b, 32 * L.W, scat_smem, s>>>(svals, cstart, rect, L.T, L.TX, L.tbits, L.nblk_b, thist,
                                                      misc + 2, sorted_idx);
  if (tile_order) k_tile_order<<<1, 1024, 0, s>>>(reinterpret_cast<const int2 *>(tile_range), L.T, tile_order);
  return check_launch("gs_bin_sort");
}
