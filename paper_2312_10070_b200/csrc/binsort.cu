// binsort.cu — S2 gs_bin_sort: tile binning with deterministic depth order
// ("m ordered Gaussians"; R10).
//
// Result = every (tile, Gaussian) pair ordered by the composite key
// (tile asc, fp32 depth asc, Gaussian id asc), computed as two stable LSD
// radix sorts that together equal one sort on that key:
//   1. the Gaussians by depth bits (z_near-relative, 9-bit digits; invisible
//      Gaussians get an all-ones key and land after the Nv visible ones; the
//      input order is the Gaussian id, so equal depths stay in id order);
//   2. the (tile, depth rank) pairs, emitted in depth-rank order, by the tile
//      bits only (7-bit digits): stability keeps rank (= depth, id) order
//      inside every tile.
// Every radix pass is ONE "onesweep" kernel: blocks take tickets in launch
// order, rank their keys per warp with ballot-sliced peer masks (MATCH.ANY is
// ~100x slower on this part), publish per-digit block counts and find their
// global offsets by decoupled look-back over the preceding blocks.  The global
// digit histograms are known up front: depth digits from the prep kernel,
// tile digits from the per-tile pair counts (a 2-D difference array of the
// tile rects, 4 updates per Gaussian).  Everything is integer arithmetic: the
// output is bit-deterministic.
#include <algorithm>
#include <cstring>

#include "gs_internal.cuh"

namespace gs {

constexpr int kOSThreads = 256;  // onesweep block: 8 warps
constexpr int kDepthBits = 9;    // depth digit width
constexpr int kTileBits = 7;     // tile digit width
constexpr int kDepthItems = 8;   // keys per thread (2048 per block)
constexpr int kPairItems = 8;    // pairs per thread (2048 per block)
constexpr int kScanItems1 = 16;  // 1-pass scan: 4096 values per block
constexpr uint32_t kFlagA = 1u << 30, kFlagP = 2u << 30, kValMask = (1u << 30) - 1;
constexpr int kMaxDepthPasses = 4, kMaxTilePasses = 3;

struct SortLayout {
  int n, T, TX, TY;
  int dpasses, tpasses;
  uint32_t zbase, kinvis;
  int nblk_d, nblk_p, nblk_s;
  int64_t capacity;
  // zeroed region (one memset per call)
  size_t diff, st_s, tickets, misc, zero_end;
  // per-pass digit-major count matrices [D][nblk] (written in full by the upsweeps)
  size_t cnt_d, cnt_p, st_cd, st_cp;
  // other
  size_t dkeys_a, dkeys_b, dvals_a, dvals_b, pkeys_a, pkeys_b, pvals_a, pvals_b, total;
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static bool make_layout(int32_t n, int64_t capacity, const gs_camera &cam, SortLayout &L) {
  L.n = n;
  L.capacity = capacity;
  L.TX = tiles_x(cam);
  L.TY = tiles_y(cam);
  L.T = L.TX * L.TY;
  int tbits = 1;
  while ((1 << tbits) < L.T) ++tbits;
  L.tpasses = (tbits + kTileBits - 1) / kTileBits;
  // positive floats order as their bit patterns; keys are bits(z) - bits(z_near)
  uint32_t zb, ze;
  float zn = cam.z_near, zf = cam.z_far;
  memcpy(&zb, &zn, 4);
  memcpy(&ze, &zf, 4);
  L.zbase = zb;
  const uint64_t span = uint64_t(ze - zb) + 2;  // visible keys <= ze - zb < the all-ones key
  int bits = 1;
  while ((uint64_t(1) << bits) < span) ++bits;
  L.dpasses = (bits + kDepthBits - 1) / kDepthBits;
  if (L.dpasses > kMaxDepthPasses || L.tpasses > kMaxTilePasses || L.T > (1 << 21)) return false;
  L.kinvis = uint32_t((uint64_t(1) << (kDepthBits * L.dpasses)) - 1);
  if (capacity >= int64_t(kValMask) || int64_t(n) >= int64_t(kValMask)) return false;
  L.nblk_d = std::max(1, (n + kOSThreads * kDepthItems - 1) / (kOSThreads * kDepthItems));
  L.nblk_p = int(std::max<int64_t>(1, (capacity + kOSThreads * kPairItems - 1) / (kOSThreads * kPairItems)));
  L.nblk_s = std::max(1, (n + kOSThreads * kScanItems1 - 1) / (kOSThreads * kScanItems1));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  const size_t Dd = size_t(1) << kDepthBits, Dt = size_t(1) << kTileBits;
  const size_t ncd = Dd * L.nblk_d, ncp = Dt * L.nblk_p;
  const size_t sbd = (ncd + kOSThreads * kScanItems1 - 1) / (kOSThreads * kScanItems1);
  const size_t sbp = (ncp + kOSThreads * kScanItems1 - 1) / (kOSThreads * kScanItems1);
  L.diff = take(4 * size_t(L.TX + 1) * (L.TY + 1));
  L.st_s = take(4 * size_t(L.nblk_s));
  L.st_cd = take(4 * sbd * L.dpasses);
  L.st_cp = take(4 * sbp * L.tpasses);
  L.tickets = take(4 * 16);
  L.misc = take(64);  // [0] nvis, [1] P, [2] overflow
  L.zero_end = off;
  L.cnt_d = take(4 * ncd);
  L.cnt_p = take(4 * ncp);
  const size_t nn = size_t(n > 0 ? n : 1), cc = size_t(capacity > 0 ? capacity : 1);
  L.dkeys_a = take(4 * nn);
  L.dkeys_b = take(4 * nn);
  L.dvals_a = take(4 * nn);
  L.dvals_b = take(4 * nn);
  L.pkeys_a = take(4 * cc);
  L.pkeys_b = take(4 * cc);
  L.pvals_a = take(4 * cc);
  L.pvals_b = take(4 * cc);
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

// Lanes of `act` whose key agrees with this lane's in its low kBits bits:
// one ballot per bit.  Every lane of the warp must call it.
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

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
  return *reinterpret_cast<const volatile uint32_t *>(p);
}

__device__ __forceinline__ void st_volatile(uint32_t *p, uint32_t v) { *reinterpret_cast<volatile uint32_t *>(p) = v; }

// Decoupled look-back, one warp: publish this block's aggregate, then read the
// status words of up to 32 predecessors at once; the nearest inclusive prefix
// (flag P) ends the walk, aggregates (flag A) in front of it are added, and a
// window containing an unpublished word (0) is re-read.  Returns the
// exclusive prefix of `count` on every lane.
__device__ __forceinline__ uint32_t warp_look_back(uint32_t *status, int bid, uint32_t count) {
  const int lane = threadIdx.x & 31;
  if (bid == 0) {
    if (lane == 0) st_volatile(status, kFlagP | count);
    return 0;
  }
  if (lane == 0) st_volatile(status + bid, kFlagA | count);
  uint32_t excl = 0;
  int top = bid - 1;  // newest predecessor of the current window
  while (true) {
    const int j = top - lane;
    const uint32_t sv = j >= 0 ? ld_volatile(status + j) : kFlagP;  // virtual P before block 0
    const unsigned pmask = __ballot_sync(0xffffffffu, sv & kFlagP);
    const unsigned zmask = __ballot_sync(0xffffffffu, !(sv & (kFlagA | kFlagP)));
    const int first_p = pmask ? __ffs(pmask) - 1 : 32;
    const unsigned upto = first_p == 32 ? 0xffffffffu : (first_p == 31 ? 0xffffffffu : ((2u << first_p) - 1u));
    if (zmask & upto) continue;  // someone in front of the nearest P has not published yet
    uint32_t v = (lane <= first_p && j >= 0) ? (sv & kValMask) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (first_p < 32) break;
    top -= 32;
  }
  if (lane == 0) st_volatile(status + bid, kFlagP | (excl + count));
  return excl;
}

// ---------------------------------------------------------------------------
// Single-pass exclusive scan (in place) with decoupled look-back; total out.

__global__ void __launch_bounds__(kOSThreads) k_scan_1pass(uint32_t *a, int64_t L, uint32_t *status, uint32_t *ticket,
                                                           uint32_t *total) {
  __shared__ uint32_t sh[33];
  __shared__ uint32_t s_bid, s_prefix;
  if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
  __syncthreads();
  const int bid = int(s_bid);
  const int64_t base = int64_t(bid) * kOSThreads * kScanItems1 + int64_t(threadIdx.x) * kScanItems1;
  uint32_t v[kScanItems1];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems1; ++k) {
    v[k] = base + k < L ? a[base + k] : 0u;
    s += v[k];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan(s, sh, tot);
  if (threadIdx.x < 32) {
    const uint32_t pre = warp_look_back(status, bid, tot);
    if (threadIdx.x == 0) {
      s_prefix = pre;
      if (bid == int(gridDim.x) - 1 && total) *total = pre + tot;
    }
  }
  __syncthreads();
  ex += s_prefix;
#pragma unroll
  for (int k = 0; k < kScanItems1; ++k) {
    if (base + k < L) a[base + k] = ex;
    ex += v[k];
  }
}

// ---------------------------------------------------------------------------
// Depth prep: radix keys of all Gaussians and the tile-rect difference array
// (per-block in shared memory, merged with one global atomic per nonzero cell).

struct PrepArgs {
  const float *depth;
  const int32_t *tiles_touched;
  const short4 *rect;
  int n, TX, TY;
  uint32_t zbase, kinvis;
  uint32_t *keys, *vals, *diff, *nvis;
};

__global__ void __launch_bounds__(kOSThreads) k_depth_prep(PrepArgs a) {
  extern __shared__ uint32_t s_diff[];
  const int W1 = a.TX + 1, cells = W1 * (a.TY + 1);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) s_diff[i] = 0;
  __syncthreads();
  uint32_t vis = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
    uint32_t key = a.kinvis;
    if (__ldg(a.tiles_touched + i) > 0) {
      key = __float_as_uint(__ldg(a.depth + i)) - a.zbase;
      ++vis;
      // +1 over the rect [x0, x1] x [y0, y1]
      const short4 r = __ldg(a.rect + i);
      atomicAdd(s_diff + r.y * W1 + r.x, 1u);
      atomicAdd(s_diff + r.y * W1 + r.z + 1, 0xffffffffu);
      atomicAdd(s_diff + (r.w + 1) * W1 + r.x, 0xffffffffu);
      atomicAdd(s_diff + (r.w + 1) * W1 + r.z + 1, 1u);
    }
    a.keys[i] = key;
    a.vals[i] = uint32_t(i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vis += __shfl_xor_sync(0xffffffffu, vis, o);
  if ((threadIdx.x & 31) == 0 && vis) atomicAdd(a.nvis, vis);
  __syncthreads();
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    const uint32_t c = s_diff[i];
    if (c) atomicAdd(a.diff + i, c);
  }
}

// ---------------------------------------------------------------------------
// One stable LSD radix pass = upsweep (per-block digit counts, digit-major) +
// one-pass exclusive scan of the count matrix + downsweep (stable rank and
// scatter).  Block = 8 warps x 32 lanes x ITEMS keys; warp w owns the keys
// [base + 32 ITEMS w, +32 ITEMS), walked in ITEMS rounds of 32.

struct RSArgs {
  const uint32_t *keys_in, *vals_in;
  uint32_t *keys_out, *vals_out;
  const uint32_t *n_dev;  // element count (device), or nullptr -> n
  int64_t n;
  int shift, nblk;
  uint32_t *counts;          // [D][nblk]
  const int32_t *tiles_out;  // depth sort, last pass: write tiles_touched[val] as key
  const uint32_t *skip;      // optional flag: skip the pass when *skip != 0
};

template <int RB, int ITEMS>
__global__ void __launch_bounds__(kOSThreads) k_rs_upsweep(RSArgs a) {
  constexpr int D = 1 << RB;
  __shared__ uint32_t h[D];
  for (int d = threadIdx.x; d < D; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const bool skip = a.skip && *a.skip;
  const int64_t n = skip ? 0 : (a.n_dev ? int64_t(*a.n_dev) : a.n);
  const int64_t base = int64_t(blockIdx.x) * (kOSThreads * ITEMS);
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int64_t i = base + r * kOSThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(a.keys_in[i] >> a.shift) & (D - 1)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x) a.counts[size_t(d) * a.nblk + blockIdx.x] = h[d];
}

template <int RB, int ITEMS>
__global__ void __launch_bounds__(kOSThreads) k_rs_downsweep(RSArgs a) {
  constexpr int D = 1 << RB, W = kOSThreads / 32;
  __shared__ uint32_t s_wc[W][D];
  if (a.skip && *a.skip) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < W * D; i += blockDim.x) (&s_wc[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = a.n_dev ? int64_t(*a.n_dev) : a.n;
  const int64_t base = int64_t(blockIdx.x) * (kOSThreads * ITEMS) + int64_t(w) * (32 * ITEMS);
  uint32_t key[ITEMS], val[ITEMS], rank[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int64_t i = base + r * 32 + lane;
    key[r] = i < n ? a.keys_in[i] : 0xffffffffu;
    val[r] = i < n ? a.vals_in[i] : 0u;
  }
  // per-warp stable ranks (rounds in input order, lanes in input order)
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const bool ok = base + r * 32 + lane < n;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    const uint32_t d = (key[r] >> a.shift) & (D - 1);
    const unsigned peers = peer_mask<RB>(act, d);
    const uint32_t before = ok ? s_wc[w][d] : 0u;
    rank[r] = before + __popc(peers & lanemask_lt());
    __syncwarp();
    if (ok && lane == 31 - __clz(peers)) s_wc[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive warp prefixes + the block's global offset
  for (int d = threadIdx.x; d < D; d += kOSThreads) {
    uint32_t run = a.counts[size_t(d) * a.nblk + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < W; ++ww) {
      const uint32_t c = s_wc[ww][d];
      s_wc[ww][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    if (base + r * 32 + lane >= n) continue;
    const uint32_t d = (key[r] >> a.shift) & (D - 1);
    const uint32_t pos = s_wc[w][d] + rank[r];
    a.keys_out[pos] = a.tiles_out ? uint32_t(__ldg(a.tiles_out + val[r])) : key[r];
    a.vals_out[pos] = val[r];
  }
}

// ---------------------------------------------------------------------------
// Per-tile pair counts (2-D prefix of the difference array, in shared
// memory), tile ranges, P and the capacity check, heaviest-first tile order.

struct TileArgs {
  const uint32_t *diff;  // (TY+1) x (TX+1)
  int TX, TY, T;
  int64_t capacity;
  int32_t *tile_range, *tile_order;
  int64_t *n_pairs;
  uint32_t *misc;  // [1] P, [2] overflow
  gs_counters *cnt;
};

__global__ void __launch_bounds__(1024) k_tile_counts(TileArgs a) {
  extern __shared__ uint32_t s_c[];  // (TY+1) x (TX+1)
  __shared__ uint32_t sh[33];
  __shared__ int s_max;
  __shared__ unsigned s_b[64];
  const int W1 = a.TX + 1, cells = W1 * (a.TY + 1);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) s_c[i] = a.diff[i];
  if (threadIdx.x == 0) s_max = 0;
  if (threadIdx.x < 64) s_b[threadIdx.x] = 0;
  __syncthreads();
  // rows, then columns: diff -> per-tile counts
  for (int y = threadIdx.x; y < a.TY; y += blockDim.x) {
    uint32_t run = 0;
    for (int x = 0; x < a.TX; ++x) {
      run += s_c[y * W1 + x];
      s_c[y * W1 + x] = run;
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < a.TX; x += blockDim.x) {
    uint32_t run = 0;
    for (int y = 0; y < a.TY; ++y) {
      run += s_c[y * W1 + x];
      s_c[y * W1 + x] = run;
    }
  }
  __syncthreads();
  // exclusive scan over tiles (tile id = y*TX + x), PER consecutive tiles per thread
  const int PER = (a.T + blockDim.x - 1) / blockDim.x;
  uint32_t s = 0;
  int m = 0;
  for (int k = 0; k < PER; ++k) {
    const int t = threadIdx.x * PER + k;
    if (t < a.T) {
      const uint32_t c = s_c[(t / a.TX) * W1 + t % a.TX];
      s += c;
      m = max(m, int(c));
    }
  }
  uint32_t P;
  uint32_t ex = block_excl_scan(s, sh, P);
  const bool over = int64_t(P) > a.capacity;
  atomicMax(&s_max, m);
  for (int k = 0; k < PER; ++k) {
    const int t = threadIdx.x * PER + k;
    if (t < a.T) {
      const uint32_t c = s_c[(t / a.TX) * W1 + t % a.TX];
      reinterpret_cast<int2 *>(a.tile_range)[t] = over ? make_int2(0, 0) : make_int2(int(ex), int(ex + c));
      ex += c;
    }
  }
  if (threadIdx.x == 0) {
    a.misc[1] = P;
    a.misc[2] = over ? 1u : 0u;
    *a.n_pairs = int64_t(P);
    if (over && a.cnt) atomicAdd(reinterpret_cast<unsigned long long *>(&a.cnt->n_overflow), 1ull);
  }
  if (!a.tile_order) return;
  __syncthreads();
  // heaviest first: 64 buckets of maxlen/64 (order inside a bucket unspecified)
  const int den = s_max + 1;
  for (int t = threadIdx.x; t < a.T; t += blockDim.x) {
    const uint32_t c = s_c[(t / a.TX) * W1 + t % a.TX];
    atomicAdd(&s_b[63 - int((int64_t(c) * 64) / den)], 1u);
  }
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
  for (int t = threadIdx.x; t < a.T; t += blockDim.x) {
    const uint32_t c = s_c[(t / a.TX) * W1 + t % a.TX];
    a.tile_order[atomicAdd(&s_b[63 - int((int64_t(c) * 64) / den)], 1u)] = t;
  }
}

// ---------------------------------------------------------------------------
// Pair emission in depth-rank order: one item per warp step, lanes = its tiles.

__global__ void __launch_bounds__(kOSThreads) k_emit_pairs(const uint32_t *__restrict__ svals,
                                                           const uint32_t *__restrict__ poff,
                                                           const short4 *__restrict__ rect,
                                                           const uint32_t *__restrict__ nvis,
                                                           const uint32_t *__restrict__ overflow, int TX,
                                                           uint32_t *pkeys, uint32_t *pvals) {
  if (*overflow) return;
  const int nv = int(*nvis);
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int k0 = warp * 32;
  if (k0 >= nv) return;
  const int k = k0 + lane;
  int rxy = 0, wdt = 1, nt = 0;
  uint32_t po = 0, magic = 0;
  if (k < nv) {
    const short4 r = __ldg(rect + __ldg(svals + k));
    wdt = r.z - r.x + 1;
    nt = wdt * (r.w - r.y + 1);
    rxy = (int(r.x) & 0xffff) | (int(r.y) << 16);
    po = __ldg(poff + k);
    magic = wdt > 1 ? uint32_t((0x100000000ull + uint64_t(wdt) - 1) / uint64_t(wdt)) : 0u;
  }
  const int cnt = min(32, nv - k0);
  for (int i = 0; i < cnt; ++i) {
    const int ixy = __shfl_sync(0xffffffffu, rxy, i);
    const int iw = __shfl_sync(0xffffffffu, wdt, i);
    const int int_ = __shfl_sync(0xffffffffu, nt, i);
    const uint32_t ipo = __shfl_sync(0xffffffffu, po, i);
    const uint32_t im = __shfl_sync(0xffffffffu, magic, i);
    const int x0 = int(short(ixy & 0xffff)), y0 = ixy >> 16;
    for (int l = lane; l < int_; l += 32) {
      const int row = iw == 1 ? l : int(__umulhi(uint32_t(l), im));  // exact for l, width < 2^16
      pkeys[ipo + l] = uint32_t((y0 + row) * TX + x0 + (l - row * iw));
      pvals[ipo + l] = uint32_t(k0 + i);
    }
  }
}

// sorted_idx[p] = Gaussian of the p-th pair (rank -> id through the depth sort).
__global__ void __launch_bounds__(256) k_gather_ids(const uint32_t *__restrict__ prank,
                                                    const uint32_t *__restrict__ svals,
                                                    const uint32_t *__restrict__ misc, int32_t *sorted_idx) {
  if (misc[2]) return;
  const int64_t P = misc[1];
  const int64_t p0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (p0 + 3 < P) {
    const uint4 r = __ldg(reinterpret_cast<const uint4 *>(prank + p0));
    int4 o;
    o.x = int32_t(__ldg(svals + r.x));
    o.y = int32_t(__ldg(svals + r.y));
    o.z = int32_t(__ldg(svals + r.z));
    o.w = int32_t(__ldg(svals + r.w));
    *reinterpret_cast<int4 *>(sorted_idx + p0) = o;
  } else {
    for (int64_t p = p0; p < P && p < p0 + 4; ++p) sorted_idx[p] = int32_t(__ldg(svals + __ldg(prank + p)));
  }
}

}  // namespace gs

namespace gs {
// Tiles by descending work, 64 buckets of max/64 (single CTA).
__global__ void __launch_bounds__(1024) k_order_by_work(const int32_t *__restrict__ work, int T, int32_t *order) {
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
  k_order_by_work<<<1, 1024, 0, as_stream(stream)>>>(work, T, order);
  return check_launch("gs_tile_order");
}

extern "C" size_t gs_binsort_workspace_bytes(int32_t n, int64_t capacity, gs_camera cam) {
  gs::SortLayout L;
  if (n < 0 || capacity < 0 || !gs::camera_ok(cam) || !gs::make_layout(n, capacity, cam, L)) return 0;
  return L.total;
}

namespace gs {
template <int RB, int ITEMS>
static void radix_pass(const RSArgs &a, uint32_t *scan_status, uint32_t *ticket, cudaStream_t s) {
  const int64_t L = int64_t(1 << RB) * a.nblk;
  k_rs_upsweep<RB, ITEMS><<<a.nblk, kOSThreads, 0, s>>>(a);
  const int nb = int((L + kOSThreads * kScanItems1 - 1) / (kOSThreads * kScanItems1));
  k_scan_1pass<<<nb, kOSThreads, 0, s>>>(a.counts, L, scan_status, ticket, nullptr);
  k_rs_downsweep<RB, ITEMS><<<a.nblk, kOSThreads, 0, s>>>(a);
}
}  // namespace gs

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
  if (!make_layout(n, capacity, cam, L)) {
    set_error("gs_bin_sort: problem too large (n=%d, capacity=%lld, tiles=%d)", n, (long long)capacity,
              tiles_x(cam) * tiles_y(cam));
    return GS_ERR_UNSUPPORTED;
  }
  if (!ws || ws_bytes < L.total) {
    set_error("gs_bin_sort: workspace %zu < %zu bytes", ws_bytes, L.total);
    return GS_ERR_WORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  char *w = static_cast<char *>(ws);
  auto U = [&](size_t off) { return reinterpret_cast<uint32_t *>(w + off); };
  uint32_t *misc = U(L.misc), *tickets = U(L.tickets);
  cudaMemsetAsync(w, 0, L.zero_end, s);
  const short4 *rect = reinterpret_cast<const short4 *>(pr.rect);
  const size_t diff_bytes = size_t(4) * (L.TX + 1) * (L.TY + 1);
  static thread_local size_t smem_set = 0;
  if (diff_bytes > 48 * 1024 && diff_bytes > smem_set) {
    cudaFuncSetAttribute(k_depth_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, int(diff_bytes));
    cudaFuncSetAttribute(k_tile_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, int(diff_bytes));
    smem_set = diff_bytes;
  }
  // ---- depth keys, tile difference array, per-tile pair counts ----
  {
    PrepArgs a{pr.depth, pr.tiles_touched, rect, n, L.TX, L.TY, L.zbase, L.kinvis,
               U(L.dkeys_a), U(L.dvals_a), U(L.diff), misc + 0};
    const int blocks = std::max(1, std::min(2 * 148, (n + kOSThreads - 1) / kOSThreads));
    k_depth_prep<<<blocks, kOSThreads, diff_bytes, s>>>(a);
  }
  {
    TileArgs a{U(L.diff), L.TX, L.TY, L.T, capacity, tile_range, tile_order, n_pairs, misc, cnt};
    k_tile_counts<<<1, 1024, diff_bytes, s>>>(a);
  }
  // ---- stage 1: depth radix passes (last pass writes tiles_touched[val]) ----
  uint32_t *dk[2] = {U(L.dkeys_a), U(L.dkeys_b)}, *dv[2] = {U(L.dvals_a), U(L.dvals_b)};
  const size_t sbd = (size_t(1 << kDepthBits) * L.nblk_d + kOSThreads * kScanItems1 - 1) / (kOSThreads * kScanItems1);
  const size_t sbp = (size_t(1 << kTileBits) * L.nblk_p + kOSThreads * kScanItems1 - 1) / (kOSThreads * kScanItems1);
  int cur = 0;
  for (int p = 0; p < L.dpasses; ++p) {
    const bool last = p == L.dpasses - 1;
    RSArgs a{dk[cur], dv[cur], dk[cur ^ 1], dv[cur ^ 1], nullptr, n, p * kDepthBits, L.nblk_d, U(L.cnt_d),
             last ? pr.tiles_touched : nullptr, nullptr};
    radix_pass<kDepthBits, kDepthItems>(a, U(L.st_cd) + p * sbd, tickets + p, s);
    cur ^= 1;
  }
  uint32_t *svals = dv[cur], *poff = dk[cur];
  // ---- pair offsets of the depth-sorted stream, pair emission ----
  k_scan_1pass<<<L.nblk_s, kOSThreads, 0, s>>>(poff, n, U(L.st_s), tickets + 8, nullptr);
  {
    const int blocks = std::max(1, (n + kOSThreads - 1) / kOSThreads);
    k_emit_pairs<<<blocks, kOSThreads, 0, s>>>(svals, poff, rect, misc + 0, misc + 2, L.TX, U(L.pkeys_a),
                                               U(L.pvals_a));
  }
  // ---- stage 2: stable tile radix passes over the pairs ----
  uint32_t *pk[2] = {U(L.pkeys_a), U(L.pkeys_b)}, *pv[2] = {U(L.pvals_a), U(L.pvals_b)};
  int pc = 0;
  for (int p = 0; p < L.tpasses; ++p) {
    RSArgs a{pk[pc], pv[pc], pk[pc ^ 1], pv[pc ^ 1], misc + 1, capacity, p * kTileBits, L.nblk_p, U(L.cnt_p),
             nullptr, misc + 2};
    radix_pass<kTileBits, kPairItems>(a, U(L.st_cp) + p * sbp, tickets + 4 + p, s);
    pc ^= 1;
  }
  if (capacity > 0) {
    const int blocks = int((capacity + 1023) / 1024);
    k_gather_ids<<<blocks, 256, 0, s>>>(pv[pc], svals, misc, sorted_idx);
  }
  return check_launch("gs_bin_sort");
}
