// binsort.cu — S2 gs_bin_sort: tile binning with deterministic depth order
// ("m ordered Gaussians"; R10).
//
// Result = every (tile, Gaussian) pair ordered by the composite key
// (tile asc, fp32 depth asc, Gaussian id asc).  Built tile by tile, with no
// global sort and no pass whose blocks wait on each other:
//   1. k_bin_prep: per-tile pair counts from a 2-D difference array of the
//      tile rects (4 shared-memory updates per visible Gaussian, merged into
//      one global array per block);
//   2. k_tile_counts (one CTA): 2-D prefix -> counts -> tile ranges (scan),
//      the capacity check, per-tile write cursors and the heaviest-first
//      launch order; without a requested order, k_tile_rows instead (one CTA
//      per tile row, closed-form row offsets, no inter-CTA communication);
//   3. k_emit: every visible Gaussian appends its id to the segment of each
//      tile of its rect (block-aggregated: shared-memory counts, one global
//      cursor reservation per (block, tile), warp-balanced pair expansion);
//      the order inside a segment is arbitrary at this point;
//   4. k_tile_sort (k_tile_sort_p: persistent CTAs taking tiles from a
//      counter, loads pipelined across tiles) sorts a segment in shared memory in
//      one pass: a counting sort on the top 10 (lists <= 2048) or 11 bits
//      of (depth bits - tile minimum), then every entry ranked inside its
//      bucket on the exact key (depth bits, id).  Segments longer than 4096
//      entries, or with a bucket of more than 128 (a dense cluster of depths
//      next to a far outlier), are left to k_tile_sort_big: an exact two-key
//      stable LSD radix sort (id digits, then depth digits; 9-bit digits,
//      warp ranks from ballot-sliced peer masks) chunk by chunk over global
//      memory.
// Everything is integer arithmetic on the fp32 depth bits (positive floats
// order as their bit patterns): the output is bit-deterministic whatever the
// order of the atomics in step 3.
#include <algorithm>
#include <cstring>

#include "gs_internal.cuh"

namespace gs {

constexpr int kSortThreads = 256;  // k_tile_sort CTA: 8 warps
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;                          // keys per thread
constexpr int kChunk = kSortThreads * kSortItems;       // 4096 keys sorted in shared memory at once
constexpr int kDigitBits = 9;
constexpr int kDigits = 1 << kDigitBits;
#ifndef TS_THREADS
#define TS_THREADS 256
#endif
constexpr int kBucketThreads = TS_THREADS;  // k_tile_sort CTA
constexpr int kMaxBucket = 128;     // fuller buckets -> exact two-key sort (k_tile_sort_big)
#ifndef EMIT_THREADS
#define EMIT_THREADS 512
#endif
constexpr int kEmitThreads = EMIT_THREADS;
// grids: the emission takes the fewest Gaussians per thread (1, 2, 4, 8) that
// keep it within EMIT_WAVES CTAs per SM, the prep at most PREP_WAVES CTAs per
// SM (each merges a full difference array with global atomics); measured
// (3, 1) against (2, 2): 2458 -> 2472 MP/s, 2821 -> 2841 it/s
#ifndef EMIT_WAVES
#define EMIT_WAVES 3
#endif
#ifndef TILE_ROWS
#define TILE_ROWS 1
#endif
#ifndef PREP_WAVES
#define PREP_WAVES 1
#endif
constexpr int kBigBlocks = 148;    // k_tile_sort_big grid (grid-stride over the long tiles)

struct SortLayout {
  int n, T, TX, TY;
  int64_t capacity;
  size_t diff, misc, zero_end;  // zeroed region (one memset per call)
  size_t cursor, slow, mid, key_a, key_b, val_b, total;
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static bool make_layout(int32_t n, int64_t capacity, const gs_camera &cam, SortLayout &L) {
  L.n = n;
  L.capacity = capacity;
  L.TX = tiles_x(cam);
  L.TY = tiles_y(cam);
  L.T = L.TX * L.TY;
  if (L.T > (1 << 21) || capacity >= (int64_t(1) << 31) - 1) return false;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  L.diff = take(4 * size_t(L.TX + 1) * (L.TY + 1));
  L.misc = take(64);  // [1] P, [2] overflow, [3] slow-list length, [4] mid-list length
  L.zero_end = off;
  L.cursor = take(4 * size_t(L.T));
  L.slow = take(4 * size_t(L.T));
  L.mid = take(4 * size_t(L.T));
  const size_t cc = size_t(capacity > 0 ? capacity : 1);
  L.key_a = take(4 * cc);  // scratch of the chunked (long-segment) sort
  L.key_b = take(4 * cc);
  L.val_b = take(4 * cc);
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

// In-place 2-D inclusive prefix (rows, then columns) of the TX x TY corner of
// a shared (TY+1) x W1 difference array: per-tile counts.  One warp per row /
// column, 32 elements per step (warp scan + carry).
__device__ void prefix2d(uint32_t *c, int W1, int TX, int TY) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int y = w; y < TY; y += nw) {
    uint32_t carry = 0;
    for (int x0 = 0; x0 < TX; x0 += 32) {
      const int x = x0 + lane;
      const uint32_t inc = warp_incl_scan(x < TX ? c[y * W1 + x] : 0u) + carry;
      if (x < TX) c[y * W1 + x] = inc;
      carry = __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
  for (int x = w; x < TX; x += nw) {
    uint32_t carry = 0;
    for (int y0 = 0; y0 < TY; y0 += 32) {
      const int y = y0 + lane;
      const uint32_t inc = warp_incl_scan(y < TY ? c[y * W1 + x] : 0u) + carry;
      if (y < TY) c[y * W1 + x] = inc;
      carry = __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
}

// Lanes of `act` whose digit equals this lane's: one ballot per digit bit.
// Every lane of the warp must call it.
__device__ __forceinline__ unsigned peer_mask(unsigned act, uint32_t d) {
  unsigned m = act;
#pragma unroll
  for (int b = 0; b < kDigitBits; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned bb = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bb : ~bb;
  }
  return m;
}

// floor(c * 64 / den) for c < 2^25, den >= 1, exact: a float estimate
// corrected by one step (no 64-bit integer division on the hot path)
__device__ __forceinline__ int bucket64(uint32_t c, uint32_t den, float inv_den) {
  const uint32_t x = c * 64u;
  int q = int(float(x) * inv_den);
  if (uint64_t(q) * den > x) --q;
  else if (uint64_t(q + 1) * den <= x) ++q;
  return q;
}

// tile row t / TX for t < 2^22, TX < 2^12: floor((t + 0.5) / TX) in fp32 is exact
__device__ __forceinline__ int tile_row(int t, float inv_tx) { return int((float(t) + 0.5f) * inv_tx); }

// ---------------------------------------------------------------------------
// Step 1: tile-rect difference array (per-block in shared memory, merged with
// one global atomic per nonzero cell).

__global__ void __launch_bounds__(256) k_bin_prep(const int32_t *__restrict__ tiles_touched,
                                                  const short4 *__restrict__ rect, int n, int TX, int TY,
                                                  uint32_t *diff) {
  pdl_begin();
  extern __shared__ uint32_t s_diff[];
  const int W1 = TX + 1, cells = W1 * (TY + 1);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) s_diff[i] = 0;
  __syncthreads();
  // kPrepPer Gaussians per thread and round, every load issued before the
  // first use (the rect is loaded whatever tiles_touched says: no dependent
  // second round trip)
  constexpr int kPrepPer = 8;
  const int stride = gridDim.x * blockDim.x;
  for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += kPrepPer * stride) {
    int tt[kPrepPer];
    short4 r[kPrepPer];
#pragma unroll
    for (int k = 0; k < kPrepPer; ++k) {
      const int i = i0 + k * stride;
      tt[k] = i < n ? __ldg(tiles_touched + i) : 0;
      r[k] = i < n ? __ldg(rect + i) : make_short4(0, 0, -1, -1);
    }
#pragma unroll
    for (int k = 0; k < kPrepPer; ++k) {
      if (tt[k] > 0) {  // +1 over the rect [x0, x1] x [y0, y1]
        atomicAdd(s_diff + r[k].y * W1 + r[k].x, 1u);
        atomicAdd(s_diff + r[k].y * W1 + r[k].z + 1, 0xffffffffu);
        atomicAdd(s_diff + (r[k].w + 1) * W1 + r[k].x, 0xffffffffu);
        atomicAdd(s_diff + (r[k].w + 1) * W1 + r[k].z + 1, 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cells; i += blockDim.x) {
    const uint32_t c = s_diff[i];
    if (c) atomicAdd(diff + i, c);
  }
}

// ---------------------------------------------------------------------------
// Step 2: per-tile pair counts (2-D prefix of the difference array, in shared
// memory), tile ranges, write cursors, P and the capacity check,
// heaviest-first tile order.

struct TileArgs {
  const uint32_t *diff;  // (TY+1) x (TX+1)
  int TX, TY, T;
  int64_t capacity;
  int32_t *tile_range, *tile_order;
  uint32_t *cursor;
  int64_t *n_pairs;
  uint32_t *misc;  // [1] P, [2] overflow
  gs_counters *cnt;
};

__global__ void __launch_bounds__(1024) k_tile_counts(TileArgs a) {
  pdl_begin();
  extern __shared__ uint32_t s_c[];  // (TY+1) x (TX+1)
  __shared__ uint32_t sh[33];
  __shared__ int s_max;
  __shared__ unsigned s_b[64];
  const int W1 = a.TX + 1, cells = W1 * (a.TY + 1);
  const float itx = 1.0f / float(a.TX);
  for (int i = threadIdx.x; i < cells; i += blockDim.x) s_c[i] = a.diff[i];
  if (threadIdx.x == 0) s_max = 0;
  if (threadIdx.x < 64) s_b[threadIdx.x] = 0;
  __syncthreads();
  prefix2d(s_c, W1, a.TX, a.TY);  // diff -> per-tile counts
  // exclusive scan over tiles (tile id = y*TX + x), PER consecutive tiles per thread
  const int PER = (a.T + blockDim.x - 1) / blockDim.x;
  uint32_t s = 0;
  int m = 0;
  for (int k = 0; k < PER; ++k) {
    const int t = threadIdx.x * PER + k;
    if (t < a.T) {
      const uint32_t c = s_c[t + tile_row(t, itx)];  // (t / TX) W1 + t % TX
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
      const uint32_t c = s_c[t + tile_row(t, itx)];  // (t / TX) W1 + t % TX
      reinterpret_cast<int2 *>(a.tile_range)[t] = over ? make_int2(0, 0) : make_int2(int(ex), int(ex + c));
      a.cursor[t] = ex;
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
  const uint32_t den = uint32_t(s_max) + 1u;
  const float iden = 1.0f / float(den);
  for (int t = threadIdx.x; t < a.T; t += blockDim.x) {
    const uint32_t c = s_c[t + tile_row(t, itx)];  // (t / TX) W1 + t % TX
    atomicAdd(&s_b[63 - bucket64(c, den, iden)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the 64 buckets (2 per lane)
    const unsigned b0 = s_b[2 * threadIdx.x], b1 = s_b[2 * threadIdx.x + 1];
    const unsigned ex = warp_incl_scan(b0 + b1) - b0 - b1;
    s_b[2 * threadIdx.x] = ex;
    s_b[2 * threadIdx.x + 1] = ex + b0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < a.T; t += blockDim.x) {
    const uint32_t c = s_c[t + tile_row(t, itx)];  // (t / TX) W1 + t % TX
    a.tile_order[atomicAdd(&s_b[63 - bucket64(c, den, iden)], 1u)] = t;
  }
}

// Step 2 without the heaviest-first order (what the pipelines request): one
// CTA per tile row y and no communication between CTAs.  With d the
// difference array (its extra row and column ignored) and, per column x',
//   col_y(x') = sum_{y'' <= y} d(x', y''),  counts c(x, y) = sum_{x' <= x} col_y(x'),
//   S(y) = sum_{y' < y} sum_x c(x, y') = sum_x' (TX - x') sum_{y'' < y} (y - y'') d(x', y''),
//   P = S(TY),
// every CTA reads the whole array (from L2), derives its row's counts, the
// pairs before its row and the total, and writes its row's ranges and
// cursors: the same values as k_tile_counts (integer arithmetic).
constexpr int kRowThreads = 128, kRowCols = 4;  // TX <= 512

__device__ __forceinline__ int block_incl_scan128(int v, int *sh, int &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int inc = int(warp_incl_scan(uint32_t(v)));
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  int before = 0;
  total = 0;
#pragma unroll
  for (int k = 0; k < kRowThreads / 32; ++k) {
    const int t = sh[k];
    before += k < w ? t : 0;
    total += t;
  }
  __syncthreads();
  return before + inc;
}

__device__ __forceinline__ long long block_sum128(long long v, long long *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  long long t = 0;
#pragma unroll
  for (int k = 0; k < kRowThreads / 32; ++k) t += sh[k];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kRowThreads) k_tile_rows(TileArgs a) {
  pdl_begin();
  __shared__ int s_sc[kRowThreads / 32];
  __shared__ long long s_ll[kRowThreads / 32];
  const int y = blockIdx.x, W1 = a.TX + 1;
  int col[kRowCols];
  long long wa = 0, wb = 0;  // sum_x' (TX - x') * (the two row-weighted column sums)
#pragma unroll
  for (int k = 0; k < kRowCols; ++k) {
    const int x = threadIdx.x + k * kRowThreads;
    int cs = 0;
    long long A = 0, B = 0;
    if (x < a.TX) {
      int yy = 0;
      for (; yy + 16 <= a.TY; yy += 16) {  // sixteen independent L2 loads in flight
        int d[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) d[u] = int(__ldcg(a.diff + (yy + u) * W1 + x));
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int r = yy + u;
          cs += r <= y ? d[u] : 0;
          A += r < y ? (long long)(y - r) * d[u] : 0ll;
          B += (long long)(a.TY - r) * d[u];
        }
      }
      for (; yy < a.TY; ++yy) {
        const int d = int(__ldcg(a.diff + yy * W1 + x));
        cs += yy <= y ? d : 0;
        A += yy < y ? (long long)(y - yy) * d : 0ll;
        B += (long long)(a.TY - yy) * d;
      }
      wa += (long long)(a.TX - x) * A;
      wb += (long long)(a.TX - x) * B;
    }
    col[k] = cs;
  }
  const long long S = block_sum128(wa, s_ll), P = block_sum128(wb, s_ll);
  const bool over = P > a.capacity;
  // counts c(x, y) = inclusive scan of col over x; the row's starts = their exclusive scan
  int carry_c = 0, carry_s = 0;
#pragma unroll
  for (int k = 0; k < kRowCols; ++k) {
    if (k * kRowThreads >= a.TX) break;  // block-uniform
    const int x = threadIdx.x + k * kRowThreads;
    int tot;
    const int c = block_incl_scan128(col[k], s_sc, tot) + carry_c;
    carry_c += tot;
    const int cv = x < a.TX ? c : 0;
    int tot2;
    const int incl = block_incl_scan128(cv, s_sc, tot2) + carry_s;
    carry_s += tot2;
    if (x < a.TX) {
      const int t = y * a.TX + x;
      const long long start = S + (incl - cv);
      reinterpret_cast<int2 *>(a.tile_range)[t] = over ? make_int2(0, 0) : make_int2(int(start), int(start + cv));
      a.cursor[t] = uint32_t(start);
    }
  }
  if (y == 0 && threadIdx.x == 0) {
    a.misc[1] = uint32_t(P);
    a.misc[2] = over ? 1u : 0u;
    *a.n_pairs = P;
    if (over && a.cnt) atomicAdd(reinterpret_cast<unsigned long long *>(&a.cnt->n_overflow), 1ull);
  }
}

// ---------------------------------------------------------------------------
// Step 3: pair emission into the tile segments (unordered inside a segment).
// Per block of kEmitThreads * kEmitPer Gaussians: the block's per-tile counts
// from a shared-memory 2-D difference array (4 updates per Gaussian), one
// global cursor reservation per (block, tile), then the pairs: every warp
// expands the rects of 32 Gaussians into one flat list of (Gaussian, tile)
// pairs walked 32 at a time (a lane finds its Gaussian by a binary search of
// the warp's inclusive prefix of tile counts), so lanes stay busy whatever
// the mix of rect sizes.

template <int kEmitPer>  // Gaussians per thread
__global__ void __launch_bounds__(kEmitThreads) k_emit(const int32_t *__restrict__ tiles_touched,
                                                       const short4 *__restrict__ rect, int n, int TX, int TY,
                                                       uint32_t *cursor, const uint32_t *__restrict__ misc,
                                                       int32_t *ids) {
  pdl_begin();
  extern __shared__ uint32_t s_e[];  // [(TY+1)(TX+1)] diff -> counts -> cursors, [T] bases
  if (misc[2]) return;               // overflow: leave sorted_idx untouched
  const int W1 = TX + 1, cells = W1 * (TY + 1), T = TX * TY;
  const float itx = 1.0f / float(TX);
  uint32_t *s_cur = s_e, *s_base = s_e + cells;
  const int lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < cells; c += blockDim.x) s_cur[c] = 0;
  __syncthreads();
  short4 r[kEmitPer];
#pragma unroll
  for (int k = 0; k < kEmitPer; ++k) {
    const int i = (blockIdx.x * kEmitPer + k) * kEmitThreads + threadIdx.x;
    const bool vis = i < n && __ldg(tiles_touched + i) > 0;
    const short4 ri = i < n ? __ldg(rect + i) : make_short4(0, 0, -1, -1);  // not behind the visibility load
    r[k] = vis ? ri : make_short4(0, 0, -1, -1);
    if (vis) {
      atomicAdd(s_cur + r[k].y * W1 + r[k].x, 1u);
      atomicAdd(s_cur + r[k].y * W1 + r[k].z + 1, 0xffffffffu);
      atomicAdd(s_cur + (r[k].w + 1) * W1 + r[k].x, 0xffffffffu);
      atomicAdd(s_cur + (r[k].w + 1) * W1 + r[k].z + 1, 1u);
    }
  }
  __syncthreads();
  prefix2d(s_cur, W1, TX, TY);
  // one reservation per (block, tile); four independent atomics in flight per thread
  for (int t0 = threadIdx.x; t0 < T; t0 += 4 * blockDim.x) {
    uint32_t cnt[4], base[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * blockDim.x;
      cnt[u] = t < T ? s_cur[t + tile_row(t, itx)] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) base[u] = cnt[u] ? atomicAdd(cursor + t0 + u * blockDim.x, cnt[u]) : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * blockDim.x;
      if (t < T) {
        s_base[t] = base[u];
        s_cur[t + tile_row(t, itx)] = 0;
      }
    }
  }
  __syncthreads();
  // the pairs: per warp round of 32 Gaussians (one per lane), the flat list of
  // their tiles (lane-major, row-major inside a rect) walked 32 slots per step.
  // The owner of slot p is the r-th Gaussian with tiles, r = (Gaussians started
  // by the step's first slot) - 1 + (starts inside (p0, p]): a ballot, one OR
  // reduction of the start bits and a popcount, then a lookup of r's lane
  // (no dependent chain of shuffles as in a binary search).
  __shared__ unsigned char s_own[kEmitThreads / 32][32];
  unsigned char *own = s_own[threadIdx.x >> 5];
#pragma unroll
  for (int k = 0; k < kEmitPer; ++k) {
    const int i = (blockIdx.x * kEmitPer + k) * kEmitThreads + threadIdx.x;
    const int wdt = r[k].z - r[k].x + 1;
    const int nt = wdt * (r[k].w - r[k].y + 1);  // 0 when not visible
    const int incl = int(warp_incl_scan(uint32_t(nt)));
    const int excl = incl - nt;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int xy = (int(r[k].x) & 0xffff) | (int(r[k].y) << 16);
    // row = floor(local / wdt) as floor((local + 0.5) (1 / wdt)) in fp32: exact
    // (local < 2^22, wdt < 2^12: the quotient is >= 0.5 / wdt from an integer)
    const float iw = 1.0f / float(max(wdt, 1));
    const bool has = nt > 0;
    const unsigned hm = __ballot_sync(0xffffffffu, has);
    __syncwarp();  // the previous round's lookups are done
    if (has) own[__popc(hm & lanemask_lt())] = (unsigned char)lane;
    __syncwarp();
    for (int p0 = 0; p0 < total; p0 += 32) {
      const int p = p0 + lane;
      const int c0 = __popc(__ballot_sync(0xffffffffu, has && excl <= p0));
      const unsigned M = __reduce_or_sync(0xffffffffu, (has && excl > p0 && excl < p0 + 32) ? 1u << (excl - p0) : 0u);
      const int rank = min(c0 - 1 + __popc(M & (0xffffffffu >> (31 - lane))), 31);
      const int j = own[rank];
      const int ej = __shfl_sync(0xffffffffu, excl, j);
      const int wj = __shfl_sync(0xffffffffu, wdt, j), xyj = __shfl_sync(0xffffffffu, xy, j);
      const float iwj = __shfl_sync(0xffffffffu, iw, j);
      if (p < total) {
        const int local = p - ej;
        const int row = int((float(local) + 0.5f) * iwj);
        const int col = local - row * wj;
        const int x = (xyj & 0xffff) + col, y = (xyj >> 16) + row;
        const uint32_t pos = s_base[y * TX + x] + atomicAdd(s_cur + y * W1 + x, 1u);
        GS_ASSERT(pos < misc[1]);  // inside the P pairs (<= capacity)
        ids[pos] = i - lane + j;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Step 4: per-tile sort.  Keys are held "blocked": warp w owns the positions
// [w*32*items, (w+1)*32*items) of the current order, its k-th round the 32
// positions w*32*items + 32k + lane.  One stable LSD pass:
//   ranks    per warp round, ballot-sliced peer masks (stable: rounds in
//            order, lanes in order) and per-warp digit counters s_cnt[w][d];
//   offsets  digit-major, warp-minor: s_off[d] (digit base) + the warps
//            before w in digit d;
//   scatter  into the shared-memory buffers, reload blocked.

struct SortSmem {
  uint32_t key[kChunk];
  uint32_t val[kChunk];
  uint16_t cnt[kSortWarps][kDigits];
  uint32_t off[kDigits];
  uint32_t sh[33];
  int flag;
  uint32_t red[3][kSortWarps];
};

// Per-warp stable ranks of the digits of one chunk; leaves the per-warp digit
// counts in s.cnt (zeroed here) and returns the ranks in rank[].
__device__ __forceinline__ void chunk_rank(const uint32_t key[kSortItems], const uint32_t val[kSortItems], int n,
                                           int items, bool by_val, int shift, SortSmem &s,
                                           uint16_t rank[kSortItems]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * kDigits / 2; i += kSortThreads)
    reinterpret_cast<uint32_t *>(&s.cnt[0][0])[i] = 0u;
  __syncthreads();
  const int base = w * 32 * items;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    if (k >= items) break;
    const bool ok = base + 32 * k + lane < n;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    const uint32_t d = ((by_val ? val[k] : key[k]) >> shift) & (kDigits - 1);
    const unsigned peers = peer_mask(act, d);
    const uint32_t before = ok ? s.cnt[w][d] : 0u;
    rank[k] = uint16_t(before + __popc(peers & lanemask_lt()));
    __syncwarp();
    if (ok && lane == 31 - __clz(peers)) s.cnt[w][d] = uint16_t(before + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
}

// s.cnt[w][d] <- sum of the counts of warps < w in digit d; returns the digit
// totals of digits 2t and 2t+1 (thread t).
__device__ __forceinline__ uint2 warp_prefix(SortSmem &s) {
  uint32_t tot[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int d = 2 * threadIdx.x + h;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = s.cnt[w][d];
      s.cnt[w][d] = uint16_t(run);
      run += c;
    }
    tot[h] = run;
  }
  return make_uint2(tot[0], tot[1]);
}

// One stable pass over a chunk held blocked in registers, scattered to
// out_key/out_val at s.off[d] + (warps before) + rank.  `local`: the chunk is
// the whole sequence, s.off = exclusive scan of its digit totals; otherwise
// s.off holds running global digit bases and is advanced by the totals.
template <bool kGlobalOut>
__device__ __forceinline__ void chunk_pass(const uint32_t key[kSortItems], const uint32_t val[kSortItems], int n,
                                           int items, bool by_val, int shift, bool local, SortSmem &s,
                                           uint32_t *out_key, uint32_t *out_val) {
  static_assert(kDigits == 2 * kSortThreads, "two digits per thread in the offset scan");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint16_t rank[kSortItems];
  chunk_rank(key, val, n, items, by_val, shift, s, rank);
  const uint2 tot = warp_prefix(s);
  if (local) {
    uint32_t all;
    const uint32_t ex = block_excl_scan(tot.x + tot.y, s.sh, all);
    s.off[2 * threadIdx.x] = ex;
    s.off[2 * threadIdx.x + 1] = ex + tot.x;
  }
  __syncthreads();
  const int base = w * 32 * items;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    if (k >= items) break;
    if (base + 32 * k + lane < n) {
      const uint32_t d = ((by_val ? val[k] : key[k]) >> shift) & (kDigits - 1);
      const uint32_t pos = s.off[d] + s.cnt[w][d] + rank[k];
      out_key[pos] = key[k];
      out_val[pos] = val[k];
    }
  }
  __syncthreads();
  if (!local) {
    s.off[2 * threadIdx.x] += tot.x;
    s.off[2 * threadIdx.x + 1] += tot.y;
    __syncthreads();
  }
}

__device__ __forceinline__ void load_blocked(uint32_t key[kSortItems], uint32_t val[kSortItems], const uint32_t *k_src,
                                             const uint32_t *v_src, int n, int items) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int base = w * 32 * items;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    if (k >= items) break;
    const int i = base + 32 * k + lane;
    key[k] = i < n ? k_src[i] : 0u;
    val[k] = i < n ? v_src[i] : 0u;
  }
}

// Bits needed for values <= x.
__device__ __forceinline__ int nbits(uint32_t x) { return x ? 32 - __clz(x) : 0; }

// Block max of three values (s.red scratch); all threads get the results.
__device__ __forceinline__ uint3 block_max3(uint3 v, SortSmem &s) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x = max(v.x, __shfl_xor_sync(0xffffffffu, v.x, o));
    v.y = max(v.y, __shfl_xor_sync(0xffffffffu, v.y, o));
    v.z = max(v.z, __shfl_xor_sync(0xffffffffu, v.z, o));
  }
  if (lane == 0) {
    s.red[0][w] = v.x;
    s.red[1][w] = v.y;
    s.red[2][w] = v.z;
  }
  __syncthreads();
  uint3 r = make_uint3(0u, 0u, 0u);
#pragma unroll
  for (int k = 0; k < kSortWarps; ++k) {
    r.x = max(r.x, s.red[0][k]);
    r.y = max(r.y, s.red[1][k]);
    r.z = max(r.z, s.red[2][k]);
  }
  __syncthreads();
  return r;
}

struct TileSortArgs {
  const float *depth;
  const int32_t *tile_range;
  const int32_t *order;  // tile launch order (nullable)
  uint32_t *misc;        // [2] overflow, [3] length of the slow-path tile list
  int T;
  int32_t *ids;  // sorted_idx
  uint32_t *key_a, *key_b, *val_b;
  int32_t *slow;  // [T] tiles left to k_tile_sort_big
  int32_t *mid;   // [T] tiles of kSmallCap+1 .. kChunk entries (k_tile_sort_mid)
};

// Tiles with <= kChunk entries, one CTA each, one pass: a counting sort on
// the top kBucketBits bits of (depth bits - tile min) into shared memory
// (positions within a bucket from shared-memory atomics, i.e. unordered),
// then every entry placed at its bucket start + the number of entries of its
// bucket with a smaller exact key (depth bits, id) (buckets hold ~n / 2048
// entries).  A tile whose buckets
// exceed kMaxBucket entries (a dense cluster of depths next to a far
// outlier), or whose list exceeds kChunk, is appended to the slow list.
// Two instances: kCap = kSmallCap (every tile, in launch order; more CTAs
// per SM: half the shared memory and registers) passes longer lists to the
// mid list, which kCap = kChunk sorts (grid-stride); longer ones, and
// dense-bucket tiles, go to the slow list.
#ifndef TS_SMALL
#define TS_SMALL 2048
#endif
#ifndef TS_SMALL_MINB
#define TS_SMALL_MINB 5
#endif
constexpr int kSmallCap = TS_SMALL;
#ifndef TS_GRID_PER_SM
#define TS_GRID_PER_SM TS_SMALL_MINB  // persistent tile-sort CTAs per SM
#endif
#ifndef TS_PERSIST
#define TS_PERSIST 1
#endif
#ifndef TS_RANK2
#define TS_RANK2 1
#endif
#ifndef TS_BUCKET_BITS
#define TS_BUCKET_BITS 10
#endif
// counting-sort buckets per tile: 2^11 for the kChunk instances, TS_BUCKET_BITS
// (2^10: measured best with bucket-order ranking) for the 2048-entry instance
template <int kCap>
constexpr int kBucketBitsOf = kCap == kSmallCap ? TS_BUCKET_BITS : 11;

template <int kCap>
struct BucketSmem {
  static constexpr int kBuckets = 1 << kBucketBitsOf<kCap>;
  alignas(16) unsigned long long comp[kCap];  // (depth bits << 32) | id: the exact composite key
  uint32_t cnt[kBuckets];         // counts, then bucket starts
  uint32_t sh[33];
  uint32_t red[2][kBucketThreads / 32];
  int flag;
};

// rank of `me` among the members [b0, be) of its bucket (the number with a
// smaller composite key); TS_RANK2: two members per 16-byte shared load
// (BJ.configs[3]: gs_bin_sort 79.3 -> 77.6 µs per view)
template <int kCap>
__device__ __forceinline__ uint32_t bucket_rank(const BucketSmem<kCap> &s, uint32_t b0, uint32_t be,
                                                unsigned long long me) {
  uint32_t rank = 0;
#if TS_RANK2
  uint32_t j = b0;
  if (j & 1u) {
    rank += s.comp[j] < me;
    ++j;
  }
  for (; j + 1 < be; j += 2) {
    const ulonglong2 c2 = *reinterpret_cast<const ulonglong2 *>(&s.comp[j]);
    rank += uint32_t(c2.x < me) + uint32_t(c2.y < me);
  }
  if (j < be) rank += s.comp[j] < me;
#else
  for (uint32_t j = b0; j < be; ++j) rank += s.comp[j] < me;
#endif
  return rank;
}

template <int kCap>
__device__ __forceinline__ bool tile_sort_one(const TileSortArgs &a, BucketSmem<kCap> &s, int tile, int2 r, int n) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int kBucketBits = kBucketBitsOf<kCap>, kBuckets = 1 << kBucketBits;
  for (int b = threadIdx.x; b < kBuckets; b += kBucketThreads) s.cnt[b] = 0u;
  if (threadIdx.x == 0) s.flag = 0;
  constexpr int kIt = kCap / kBucketThreads;
  const int items = (n + kBucketThreads - 1) / kBucketThreads;
  uint32_t key[kIt], val[kIt];
  uint32_t kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    if (k >= items) break;  // block-uniform: only the rounds this list needs
    const int i = threadIdx.x + k * kBucketThreads;
    if (i < n) {
      val[k] = uint32_t(a.ids[r.x + i]);
      key[k] = __float_as_uint(__ldg(a.depth + val[k]));
      kmin = min(kmin, key[k]);
      kmax = max(kmax, key[k]);
    }
  }
  // block min / max of the depth bits
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) {
    s.red[0][w] = kmin;
    s.red[1][w] = kmax;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < (kBucketThreads / 32); ++k) {
    kmin = min(kmin, s.red[0][k]);
    kmax = max(kmax, s.red[1][k]);
  }
  const int shift = max(0, nbits(kmax - kmin) - kBucketBits);
  uint16_t slot[kIt];
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    if (k >= items) break;  // block-uniform: only the rounds this list needs
    const int i = threadIdx.x + k * kBucketThreads;
    if (i < n) slot[k] = uint16_t(atomicAdd(&s.cnt[(key[k] - kmin) >> shift], 1u));
  }
  __syncthreads();
  // bucket starts (exclusive scan, kBuckets / kBucketThreads buckets per thread)
  constexpr int kPer = kBuckets / kBucketThreads;
  uint32_t c[kPer], sum = 0, big = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    c[k] = s.cnt[threadIdx.x * kPer + k];
    sum += c[k];
    big |= c[k] > kMaxBucket;
  }
  if (big) s.flag = 1;
  uint32_t all;
  uint32_t ex = block_excl_scan(sum, s.sh, all);
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    s.cnt[threadIdx.x * kPer + k] = ex;
    ex += c[k];
  }
  __syncthreads();
  if (s.flag) {  // dense buckets: exact two-key path
    if (threadIdx.x == 0) a.slow[atomicAdd(&a.misc[3], 1u)] = tile;
    return false;
  }
  // scatter into the buckets (unordered inside a bucket)
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    if (k >= items) break;  // block-uniform: only the rounds this list needs
    const int i = threadIdx.x + k * kBucketThreads;
    if (i < n) {
      const uint32_t pos = s.cnt[(key[k] - kmin) >> shift] + slot[k];
      s.comp[pos] = (static_cast<unsigned long long>(key[k]) << 32) | val[k];
    }
  }
  __syncthreads();
  // final position = bucket start + number of bucket entries with a smaller
  // exact key (depth bits, id): O(bucket size) per entry, no serial chain;
  // one 64-bit load and compare per member (the composite key).  Threads take
  // the entries in BUCKET order (shared-memory position), so a warp's lanes
  // share few buckets and its loop runs about as long as its own buckets
  // (numpy study at BJ.configs[3]: 4.2 members per entry against 6.6 in load
  // order, where one full bucket stalls up to that many warps)
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    if (k >= items) break;  // block-uniform: only the rounds this list needs
    const int p = threadIdx.x + k * kBucketThreads;
    if (p < n) {
      const unsigned long long me = s.comp[p];
      const uint32_t b = (uint32_t(me >> 32) - kmin) >> shift;
      const uint32_t b0 = s.cnt[b];
      const uint32_t be = b + 1 < kBuckets ? s.cnt[b + 1] : uint32_t(n);
      const uint32_t rank = bucket_rank<kCap>(s, b0, be, me);
      GS_ASSERT(int(b0 + rank) < n);
      a.ids[r.x + b0 + rank] = int32_t(uint32_t(me));
    }
  }
  return true;
}

// One CTA per tile.  kCap = kSmallCap: lists of kSmallCap+1 .. kChunk go to
// the mid list (k_tile_sort_mid); kCap = kChunk: every list <= kChunk here.
// Longer lists go to the slow list.
template <int kCap, int kMinB>
__global__ void __launch_bounds__(kBucketThreads, kMinB) k_tile_sort(TileSortArgs a) {
  pdl_begin();
  __shared__ BucketSmem<kCap> s;
  const int tile = a.order ? __ldg(a.order + blockIdx.x) : int(blockIdx.x);
  if (a.misc[2]) return;  // overflow: every range is empty
  const int2 r = reinterpret_cast<const int2 *>(a.tile_range)[tile];
  const int n = r.y - r.x;
  if (n <= 1) return;
  if (n > kCap) {  // k_tile_sort_mid / _big sort it (and mark it)
    if (threadIdx.x == 0) {
      if (n > kChunk)
        a.slow[atomicAdd(&a.misc[3], 1u)] = tile;
      else
        a.mid[atomicAdd(&a.misc[4], 1u)] = tile;
    }
    return;
  }
  tile_sort_one<kCap>(a, s, tile, r, n);
}

// Persistent variant of k_tile_sort<kSmallCap> (TS_PERSIST): CTAs take list
// positions from an atomic counter (misc[5]) and software-pipeline the global
// loads: the next position's tile range is loaded while the current tile is
// counted, its ids are loaded before the current tile's ranking phase (which
// works in shared memory only), and its depth gather opens the next round.
// One exposed global round trip per tile instead of four (order, range, ids,
// depths); same arithmetic and result as tile_sort_one.
template <int kCap, int kMinB>
__global__ void __launch_bounds__(kBucketThreads, kMinB) k_tile_sort_p(TileSortArgs a) {
  pdl_begin();
  __shared__ BucketSmem<kCap> s;
  __shared__ int s_q;
  if (a.misc[2]) return;  // overflow: every range is empty
  constexpr int kBucketBits = kBucketBitsOf<kCap>, kBuckets = 1 << kBucketBits;
  constexpr int kIt = kCap / kBucketThreads;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int2 *ranges = reinterpret_cast<const int2 *>(a.tile_range);
  if (threadIdx.x == 0) s_q = int(atomicAdd(&a.misc[5], 1u));
  __syncthreads();
  int q = s_q, tile = 0;
  int2 r = make_int2(0, 0);
  if (q < a.T) {
    tile = a.order ? __ldg(a.order + q) : q;
    r = ranges[tile];
  }
  uint32_t key[kIt], val[kIt];
  {
    const int n = r.y - r.x;
    if (n > 1 && n <= kCap) {
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        const int i = threadIdx.x + k * kBucketThreads;
        if (i < n) val[k] = uint32_t(a.ids[r.x + i]);
      }
    }
  }
  while (q < a.T) {
    __syncthreads();  // every thread has read s_q; the shared buffers are free
    if (threadIdx.x == 0) {
      s_q = int(atomicAdd(&a.misc[5], 1u));
      s.flag = 0;
    }
    const int n = r.y - r.x;
    const bool sortable = n > 1 && n <= kCap;
    if (n > kCap && threadIdx.x == 0) {  // k_tile_sort_mid / _big sort it
      if (n > kChunk)
        a.slow[atomicAdd(&a.misc[3], 1u)] = tile;
      else
        a.mid[atomicAdd(&a.misc[4], 1u)] = tile;
    }
    const int items = sortable ? (n + kBucketThreads - 1) / kBucketThreads : 0;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    for (int b = threadIdx.x; b < kBuckets; b += kBucketThreads) s.cnt[b] = 0u;
#pragma unroll
    for (int k = 0; k < kIt; ++k) {  // the depth gather of the ids loaded last round
      if (k >= items) break;
      const int i = threadIdx.x + k * kBucketThreads;
      if (i < n) {
        key[k] = __float_as_uint(__ldg(a.depth + val[k]));
        kmin = min(kmin, key[k]);
        kmax = max(kmax, key[k]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) {
      s.red[0][w] = kmin;
      s.red[1][w] = kmax;
    }
    __syncthreads();  // s_q, s.red
    // the next position's tile range (consumed after this tile's scatter)
    const int qn = s_q;
    int tile_n = 0;
    int2 r_n = make_int2(0, 0);
    if (qn < a.T) {
      tile_n = a.order ? __ldg(a.order + qn) : qn;
      r_n = ranges[tile_n];
    }
#pragma unroll
    for (int k = 0; k < (kBucketThreads / 32); ++k) {
      kmin = min(kmin, s.red[0][k]);
      kmax = max(kmax, s.red[1][k]);
    }
    const int shift = max(0, nbits(kmax - kmin) - kBucketBits);
    uint16_t slot[kIt];
#pragma unroll
    for (int k = 0; k < kIt; ++k) {
      if (k >= items) break;
      const int i = threadIdx.x + k * kBucketThreads;
      if (i < n) slot[k] = uint16_t(atomicAdd(&s.cnt[(key[k] - kmin) >> shift], 1u));
    }
    __syncthreads();
    constexpr int kPer = kBuckets / kBucketThreads;
    uint32_t c[kPer], sum = 0, big = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      c[k] = s.cnt[threadIdx.x * kPer + k];
      sum += c[k];
      big |= c[k] > kMaxBucket;
    }
    if (big && sortable) s.flag = 1;
    uint32_t all;
    uint32_t ex = block_excl_scan(sum, s.sh, all);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      s.cnt[threadIdx.x * kPer + k] = ex;
      ex += c[k];
    }
    __syncthreads();
    const bool ranked = sortable && !s.flag;
    if (sortable && s.flag && threadIdx.x == 0) a.slow[atomicAdd(&a.misc[3], 1u)] = tile;  // dense buckets
    if (ranked) {
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        if (k >= items) break;
        const int i = threadIdx.x + k * kBucketThreads;
        if (i < n) {
          const uint32_t pos = s.cnt[(key[k] - kmin) >> shift] + slot[k];
          s.comp[pos] = (static_cast<unsigned long long>(key[k]) << 32) | val[k];
        }
      }
    }
    __syncthreads();
    // the next tile's ids, in flight during this tile's ranking
    {
      const int nn = r_n.y - r_n.x;
      if (nn > 1 && nn <= kCap) {
#pragma unroll
        for (int k = 0; k < kIt; ++k) {
          const int i = threadIdx.x + k * kBucketThreads;
          if (i < nn) val[k] = uint32_t(a.ids[r_n.x + i]);
        }
      }
    }
    if (ranked) {
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        if (k >= items) break;
        const int p = threadIdx.x + k * kBucketThreads;
        if (p < n) {
          const unsigned long long me = s.comp[p];
          const uint32_t b = (uint32_t(me >> 32) - kmin) >> shift;
          const uint32_t b0 = s.cnt[b];
          const uint32_t be = b + 1 < kBuckets ? s.cnt[b + 1] : uint32_t(n);
          const uint32_t rank = bucket_rank<kCap>(s, b0, be, me);
          GS_ASSERT(int(b0 + rank) < n);
          a.ids[r.x + b0 + rank] = int32_t(uint32_t(me));
        }
      }
    }  // (a single entry is in place already)
    q = qn;
    tile = tile_n;
    r = r_n;
  }
}

__global__ void __launch_bounds__(kBucketThreads, 4) k_tile_sort_mid(TileSortArgs a) {
  pdl_begin();
  __shared__ BucketSmem<kChunk> s;
  if (a.misc[2]) return;
  const int nmid = int(a.misc[4]);
  for (int q = blockIdx.x; q < nmid; q += gridDim.x) {
    const int tile = a.mid[q];
    const int2 r = reinterpret_cast<const int2 *>(a.tile_range)[tile];
    tile_sort_one<kChunk>(a, s, tile, r, r.y - r.x);
    __syncthreads();  // the shared buffers are reused by the next tile
  }
}

// Tiles of the slow list (grid-stride): exact two-key LSD (id digits, then
// depth digits) over global memory, chunk by chunk: each chunk of kChunk
// entries ranked stably per warp round (ballot-sliced peer masks, per-warp
// digit counters), digit bases carried across chunks from a per-pass
// histogram.
__global__ void __launch_bounds__(kSortThreads) k_tile_sort_big(TileSortArgs a) {
  pdl_begin();
  __shared__ SortSmem s;
  if (a.misc[2]) return;
  const int nslow = int(a.misc[3]);
  for (int q = blockIdx.x; q < nslow; q += gridDim.x) {
    const int tile = a.slow[q];
    const int2 r = reinterpret_cast<const int2 *>(a.tile_range)[tile];
    const int n = r.y - r.x;
    uint32_t *vA = reinterpret_cast<uint32_t *>(a.ids) + r.x, *kA = a.key_a + r.x;
    uint32_t *vB = a.val_b + r.x, *kB = a.key_b + r.x;
    uint32_t kmin = 0xffffffffu, kmax = 0u, vmax = 0u;
    for (int i = threadIdx.x; i < n; i += kSortThreads) {
      const uint32_t v = vA[i];
      const uint32_t k = __float_as_uint(__ldg(a.depth + v));
      kA[i] = k;
      kmin = min(kmin, k);
      kmax = max(kmax, k);
      vmax = max(vmax, v);
    }
    const uint3 m = block_max3(make_uint3(~kmin, kmax, vmax), s);
    kmin = ~m.x;
    for (int i = threadIdx.x; i < n; i += kSortThreads) kA[i] -= kmin;
    __syncthreads();
    const int kbits = nbits(m.y - kmin), vbits = nbits(m.z);
    const int npass_v = (vbits + kDigitBits - 1) / kDigitBits, npass_k = (kbits + kDigitBits - 1) / kDigitBits;
    for (int p = 0; p < npass_v + npass_k; ++p) {
      const bool by_val = p < npass_v;
      const int shift = (by_val ? p : p - npass_v) * kDigitBits;
      // digit histogram of the whole segment -> global digit bases
      for (int d = threadIdx.x; d < kDigits; d += kSortThreads) s.off[d] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kSortThreads)
        atomicAdd(&s.off[((by_val ? vA[i] : kA[i]) >> shift) & (kDigits - 1)], 1u);
      __syncthreads();
      {
        const uint32_t c0 = s.off[2 * threadIdx.x], c1 = s.off[2 * threadIdx.x + 1];
        uint32_t all;
        const uint32_t ex = block_excl_scan(c0 + c1, s.sh, all);
        s.off[2 * threadIdx.x] = ex;
        s.off[2 * threadIdx.x + 1] = ex + c0;
        __syncthreads();
      }
      for (int c0 = 0; c0 < n; c0 += kChunk) {
        const int cn = min(kChunk, n - c0);
        const int items = (cn + kSortThreads - 1) / kSortThreads;
        uint32_t key[kSortItems], val[kSortItems];
        load_blocked(key, val, kA + c0, vA + c0, cn, items);
        chunk_pass<true>(key, val, cn, items, by_val, shift, false, s, kB, vB);
      }
      uint32_t *t0 = kA, *t1 = vA;
      kA = kB;
      vA = vB;
      kB = t0;
      vB = t1;
      __syncthreads();
    }
    uint32_t *dst = reinterpret_cast<uint32_t *>(a.ids) + r.x;
    if (vA != dst)
      for (int i = threadIdx.x; i < n; i += kSortThreads) dst[i] = vA[i];
    __syncthreads();
  }
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
  const uint32_t den = uint32_t(s_max) + 1u;
  const float iden = 1.0f / float(den);
  for (int t = threadIdx.x; t < T; t += blockDim.x) atomicAdd(&s_b[63 - bucket64(uint32_t(max(work[t], 0)), den, iden)], 1u);
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the 64 buckets (2 per lane)
    const unsigned b0 = s_b[2 * threadIdx.x], b1 = s_b[2 * threadIdx.x + 1];
    const unsigned ex = warp_incl_scan(b0 + b1) - b0 - b1;
    s_b[2 * threadIdx.x] = ex;
    s_b[2 * threadIdx.x + 1] = ex + b0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x)
    order[atomicAdd(&s_b[63 - bucket64(uint32_t(max(work[t], 0)), den, iden)], 1u)] = t;
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
  gs::SortLayout L;
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
  uint32_t *misc = U(L.misc);
  cudaMemsetAsync(w, 0, L.zero_end, s);
  const short4 *rect = reinterpret_cast<const short4 *>(pr.rect);
  const size_t diff_bytes = size_t(4) * (L.TX + 1) * (L.TY + 1);
  const size_t emit_bytes = diff_bytes + size_t(4) * L.T;
  static thread_local size_t smem_set = 0, smem_set_emit[9] = {0};
  const size_t need = std::max(diff_bytes, emit_bytes);
  if (need > 48 * 1024 && need > smem_set) {
    cudaFuncSetAttribute(k_bin_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, int(diff_bytes));
    cudaFuncSetAttribute(k_tile_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, int(diff_bytes));
    smem_set = need;
  }
  if (n > 0) {
    const int blocks = std::max(1, std::min(PREP_WAVES * 148, (n + 255) / 256));
    launch_pdl(k_bin_prep, dim3(blocks), dim3(256), diff_bytes, s, pr.tiles_touched, rect, n, L.TX, L.TY, U(L.diff));
  }
  {
    TileArgs a{U(L.diff), L.TX, L.TY, L.T, capacity, tile_range, tile_order, U(L.cursor), n_pairs, misc, cnt};
    if (TILE_ROWS && !tile_order && L.TX <= kRowThreads * kRowCols)
      launch_pdl(k_tile_rows, dim3(L.TY), dim3(kRowThreads), 0, s, a);
    else
      launch_pdl(k_tile_counts, dim3(1), dim3(1024), diff_bytes, s, a);
  }
  if (n > 0 && capacity > 0) {
    // Gaussians per thread: the smallest of 1, 2, 4, 8 that fits the grid in
    // one wave of 2 CTAs per SM (the per-CTA set-up, a 2-D prefix and one
    // cursor reservation per tile, is then paid about twice per SM)
    int per = 1;
    while (per < 8 && (n + kEmitThreads * per - 1) / (kEmitThreads * per) > EMIT_WAVES * 148) per *= 2;
    const int eb = (n + kEmitThreads * per - 1) / (kEmitThreads * per);
    auto kern = per == 1 ? k_emit<1> : per == 2 ? k_emit<2> : per == 4 ? k_emit<4> : k_emit<8>;
    if (need > 48 * 1024 && need > smem_set_emit[per]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(emit_bytes));
      smem_set_emit[per] = need;
    }
    launch_pdl(kern, dim3(eb), dim3(kEmitThreads), emit_bytes, s, pr.tiles_touched, rect, n, L.TX, L.TY,
               U(L.cursor), misc, sorted_idx);
    TileSortArgs a{pr.depth, tile_range, tile_order, misc, L.T, sorted_idx, U(L.key_a),
                   U(L.key_b), U(L.val_b), reinterpret_cast<int32_t *>(U(L.slow)),
                   reinterpret_cast<int32_t *>(U(L.mid))};
    // every list <= 2048 entries in the persistent half-size instance (more
    // CTAs per SM), longer ones (<= kChunk) on the grid-stride mid pass, the
    // rest on the exact long-list path: the same launches whatever the
    // caller's capacity (round 2: the capacity-keyed one-pass 4096-entry
    // instance for long averages is gone, BJ.configs[4] 2122 -> 2134 MP/s)
#if TS_PERSIST
    launch_pdl(k_tile_sort_p<kSmallCap, TS_SMALL_MINB>, dim3(std::min(L.T, 148 * TS_GRID_PER_SM)),
               dim3(kBucketThreads), 0, s, a);
#else
    launch_pdl(k_tile_sort<kSmallCap, TS_SMALL_MINB>, dim3(L.T), dim3(kBucketThreads), 0, s, a);
#endif
    launch_pdl(k_tile_sort_mid, dim3(std::min(L.T, 4 * kBigBlocks)), dim3(kBucketThreads), 0, s, a);
    launch_pdl(k_tile_sort_big, dim3(std::min(L.T, kBigBlocks)), dim3(kSortThreads), 0, s, a);
  }
  return check_launch("gs_bin_sort");
}
