// kernels_embed_det.cu — deterministic embedding backward (a5, deterministic mode).
//
//   dM[h1(c) + o] += lambda * g(c) * dOut[b, jZ + o]     (R15, R19)
//
// The fast path scatters with vector atomics (order unspecified).  Here every slot is summed
// in a fixed order, and only the slots some lookup touches are visited:
//   1. each (lookup b, chunk j) pair covers G = Z / A slot groups of A slots (offsets are
//      multiples of A); one item e = pair * G + i per (pair, group i), value (e << 1) | sign;
//   2. counting sort by group: per-group counts (atomics; a count is order-independent), an
//      exclusive scan gives each group's range, every item lands in its group's range (in
//      arbitrary order), then each group's items are sorted by item index (a thread per group
//      up to 32 items, CUB's segmented sort for the longer Zipf-hot groups) — so every group's
//      item order is canonical (ascending item index) whatever the timing;
//   3. a group is cut into fixed chunks of 64 items; a sub-warp (A / 4 lanes, a float4 each)
//      per chunk adds the chunk's lambda * g * dOut terms in item order; one-chunk groups add
//      straight into dM, longer ones (thousands of duplicates) leave partials that a second
//      pass adds in chunk order.
// Bitwise reproducible run to run (every order is fixed by the data, not by timing).  Work is
// O(lookups + |M| / A) (the per-group arrays), and hot rows are summed in parallel.  (Round 1
// sorted the items with a 21-bit CUB radix sort and found the groups as runs: 3 onesweep passes
// plus run detection, ~350 of the 820 us at C4; the counting sort needs no sort of the bulk.)
#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <type_traits>

#include "roast_internal.h"

namespace roast {
namespace {

// up to kDetTables tables of equal dim / chunk in one sorted pass (roast_embedding_bwd_multi):
// lookup b of the table-major batch belongs to table b / n
constexpr int kDetTables = 32;
struct DetTables {
  ModuleHash h[kDetTables];
  int64_t rows[kDetTables];
  float lam[kDetTables];
  int64_t n;   // lookups per table
};

// step 1: group of every item, its value (item << 1 | negative sign) and its arrival rank in the
// group (atomic: which item gets which rank is timing-dependent; step 2 re-sorts every group)
__global__ void emb_items_kernel(const __grid_constant__ DetTables T, const int64_t* __restrict__ idx, int64_t nlook,
                                 int q, int G, uint32_t* __restrict__ group, uint32_t* __restrict__ vals,
                                 int32_t* __restrict__ rank, int32_t* __restrict__ cnt, int32_t* err) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nlook * q) return;
  const int64_t b = p / q;
  const int j = int(p - b * q);
  const int t = int(b / T.n);
  const int64_t r = idx[b];
  if (r < 0 || r >= T.rows[t]) {   // skipped (no count, never placed); the sticky BOUNDS error is set
    atomicOr(err, 1);
    for (int i = 0; i < G; ++i) group[p * G + i] = 0xFFFFFFFFu;
    return;
  }
  const uint64_t key = uint64_t(r) * uint64_t(q) + uint64_t(j);
  const uint32_t k0 = uint32_t(T.h[t].offset(key) / T.h[t].align);
  const uint32_t neg = T.h[t].sign(key) < 0 ? 1u : 0u;
  for (int i = 0; i < G; ++i) {
    const uint32_t g = k0 + uint32_t(i);
    group[p * G + i] = g;
    vals[p * G + i] = (uint32_t(p * G + i) << 1) | neg;
    rank[p * G + i] = atomicAdd(cnt + g, 1);
  }
}

// step 2a: every item to its group's range
__global__ void emb_place_kernel(const uint32_t* __restrict__ group, const uint32_t* __restrict__ vals,
                                 const int32_t* __restrict__ rank, const int32_t* __restrict__ start, int64_t ni,
                                 uint32_t* __restrict__ sorted) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ni) return;
  const uint32_t g = group[e];
  if (g == 0xFFFFFFFFu) return;
  sorted[start[g] + rank[e]] = vals[e];
}

constexpr int kW = 64;      // items per chunk of a group's sum (fixed: the order is data-independent)
constexpr int kMedium = 256;  // groups of kSmall + 1 .. kMedium items: a warp each (longer: a CTA)
constexpr int kSmall = 16;  // groups up to this size are ordered by one thread (Poisson(6.5) at C4: 99.8 %)

// step 2b + chunk counts: a thread per group sorts a small group's items by value (= item index)
// with an insertion sort in registers; longer groups go to a list for CUB's segmented sort.
// nch = chunks of kW items (0 for an empty group), nlong = the same for multi-chunk groups only.
__global__ void emb_order_kernel(uint32_t* __restrict__ sorted, const int32_t* __restrict__ start,
                                 const int32_t* __restrict__ cnt, int64_t ngroups, int32_t* __restrict__ nch,
                                 int32_t* __restrict__ nlong, int32_t* __restrict__ seg_n,
                                 int32_t* __restrict__ seg_begin, int32_t* __restrict__ seg_end,
                                 int64_t seg_stride) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  const int n = cnt[g];
  const int b = start[g];
  const int c = (n + kW - 1) / kW;
  nch[g] = c;
  nlong[g] = c > 1 ? c : 0;
  if (n <= 1) return;
  if (n > kSmall) {   // the sort kernels take the lists in any order
    const int cls = n <= kMedium ? 0 : (n <= 4 * 256 ? 1 : 2);   // warp / CTA (4 keys per thread) / CTA (32)
    const int k = atomicAdd(seg_n + cls, 1);
    seg_begin[cls * seg_stride + k] = b;
    seg_end[cls * seg_stride + k] = b + n;
    return;
  }
  uint32_t v[kSmall];
#pragma unroll
  for (int i = 0; i < kSmall; ++i) v[i] = i < n ? sorted[b + i] : 0xFFFFFFFFu;
  // insertion sort over the fixed-size array (sentinels stay last); fully unrolled -> registers
#pragma unroll
  for (int i = 1; i < kSmall; ++i) {
#pragma unroll
    for (int k = i; k > 0; --k) {
      const uint32_t lo = min(v[k - 1], v[k]), hi = max(v[k - 1], v[k]);
      v[k - 1] = lo;
      v[k] = hi;
    }
  }
#pragma unroll
  for (int i = 0; i < kSmall; ++i)
    if (i < n) sorted[b + i] = v[i];
}

struct DetLam {   // lambda of each table and lookups per table (pass 1)
  float lam[kDetTables];
  int n;
};

// step 2b for the groups longer than kSmall (Zipf-hot rows: up to a few thousand items): a warp
// (<= kMedium items) or a CTA per group sorts its items ascending with the direction-free bitonic network (the first step of
// each merge compares i with i ^ (k - 1), then half-cleaners i ^ m), which tolerates a length
// that is not a power of two: positions >= n act as +inf and are never touched.  In shared
// memory up to kLongSmem items, in place in global memory beyond (the same network; the
// block barrier orders a block's global accesses).  Graph-capturable (no host round trip).
constexpr int kLongSmem = 8192;   // items a 256-thread CTA sorts in registers / shared memory
template <bool WARP>
__device__ __forceinline__ void bitonic_sort(uint32_t* a, int n) {
  const int tid = WARP ? int(threadIdx.x & 31) : int(threadIdx.x);
  const int nthr = WARP ? 32 : int(blockDim.x);
  int N = 1;
  while (N < n) N <<= 1;
  for (int k = 2; k <= N; k <<= 1) {
    for (int m = k >> 1; m > 0; m >>= 1) {
      for (int t = tid; t < N / 2; t += nthr) {
        // t-th pair of this step: i has bit log2(m) clear
        const int lo_bits = t & (m - 1);
        const int i = ((t - lo_bits) << 1) | lo_bits;
        const int j = m == (k >> 1) ? (i ^ (k - 1)) : (i | m);   // flip step first, then half-cleaners
        if (j < n) {
          const uint32_t x = a[i], y = a[j];
          if (x > y) {
            a[i] = y;
            a[j] = x;
          }
        }
      }
      if (WARP)
        __syncwarp();
      else
        __syncthreads();
    }
  }
}

// medium groups: one warp per group, in shared memory
__global__ void __launch_bounds__(256) emb_medsort_kernel(uint32_t* __restrict__ sorted,
                                                         const int32_t* __restrict__ seg_n,
                                                         const int32_t* __restrict__ seg_b,
                                                         const int32_t* __restrict__ seg_e) {
  __shared__ uint32_t sbuf[8][kMedium];
  uint32_t* a = sbuf[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int nseg = *seg_n;
  const int nwarps = int(gridDim.x * blockDim.x) >> 5;
  for (int k = int(blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nseg; k += nwarps) {
    const int b = seg_b[k], n = seg_e[k] - b;
    for (int i = lane; i < n; i += 32) a[i] = sorted[b + i];
    __syncwarp();
    bitonic_sort<true>(a, n);
    for (int i = lane; i < n; i += 32) sorted[b + i] = a[i];
    __syncwarp();
  }
}

// bitonic steps of distance m < kLongSmem are local to aligned kLongSmem-item tiles: run them in
// shared memory, one tile at a time (positions >= n load as +inf and are not stored back).
// full: the whole network of merges k = 2 .. kLongSmem (every tile sorted); else only the
// half-cleaners m = kLongSmem / 2 .. 1 that finish a longer merge whose first steps were global.
__device__ void bitonic_tiles_local(uint32_t* g, int n, uint32_t* tile, bool full) {
  for (int t0 = 0; t0 < n; t0 += kLongSmem) {
    for (int i = threadIdx.x; i < kLongSmem; i += blockDim.x) tile[i] = t0 + i < n ? g[t0 + i] : 0xFFFFFFFFu;
    __syncthreads();
    for (int k = full ? 2 : 2 * kLongSmem; k <= (full ? kLongSmem : 2 * kLongSmem); k <<= 1)
      for (int m = full ? (k >> 1) : (kLongSmem >> 1); m > 0; m >>= 1) {
        for (int t = threadIdx.x; t < kLongSmem / 2; t += blockDim.x) {
          const int lo_bits = t & (m - 1);
          const int i = ((t - lo_bits) << 1) | lo_bits;
          const int j = (full && m == (k >> 1)) ? (i ^ (k - 1)) : (i | m);
          const uint32_t x = tile[i], y = tile[j];
          if (x > y) {
            tile[i] = y;
            tile[j] = x;
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < kLongSmem && t0 + i < n; i += blockDim.x) g[t0 + i] = tile[i];
    __syncthreads();
  }
}

// large groups (> kMedium items): a CTA per group.  Up to kLongSmem items: CUB's block radix
// sort over the bits the item values use (6-bit digits: 4 passes at C4, instead of the ~55
// barrier-separated steps of a bitonic network for a 1000-item group).  Beyond (the hottest Zipf
// rows), the bitonic network with its tile-local steps in shared memory and only the steps of
// distance >= kLongSmem in global memory (the block barrier orders a block's global accesses).
constexpr int kLongThreads = 256;
template <int IPT, class Storage>
__device__ __forceinline__ void block_sort_segment(uint32_t* seg, int n, int end_bit, Storage& st) {
  using BlockSort = cub::BlockRadixSort<uint32_t, kLongThreads, IPT, cub::NullType, 6>;
  uint32_t keys[IPT];   // blocked arrangement; padding sorts last and is not written back
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    const int i = int(threadIdx.x) * IPT + u;
    keys[u] = i < n ? seg[i] : 0xFFFFFFFFu;
  }
  BlockSort(reinterpret_cast<typename BlockSort::TempStorage&>(st)).Sort(keys, 0, end_bit);
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    const int i = int(threadIdx.x) * IPT + u;
    if (i < n) seg[i] = keys[u];
  }
}

template <bool HUGE>
__global__ void __launch_bounds__(kLongThreads) emb_longsort_kernel(uint32_t* __restrict__ sorted,
                                                                   const int32_t* __restrict__ seg_n,
                                                                   const int32_t* __restrict__ seg_b,
                                                                   const int32_t* __restrict__ seg_e, int end_bit) {
  using S4 = cub::BlockRadixSort<uint32_t, kLongThreads, 4, cub::NullType, 6>;
  using S32 = cub::BlockRadixSort<uint32_t, kLongThreads, kLongSmem / kLongThreads, cub::NullType, 6>;
  __shared__ union {
    typename std::conditional<HUGE, typename S32::TempStorage, typename S4::TempStorage>::type sort;
    uint32_t tile[HUGE ? kLongSmem : 1];
  } sm;
  const int nseg = *seg_n;
  for (int k = blockIdx.x; k < nseg; k += gridDim.x) {
    const int b = seg_b[k], n = seg_e[k] - b;
    if (!HUGE) {                           // <= 4 * kLongThreads items: 4 keys per thread
      block_sort_segment<4>(sorted + b, n, end_bit, sm.sort);
    } else if (n <= kLongSmem) {
      block_sort_segment<kLongSmem / kLongThreads>(sorted + b, n, end_bit, sm.sort);
    } else {
      uint32_t* g = sorted + b;
      int N = 1;
      while (N < n) N <<= 1;
      bitonic_tiles_local(g, n, sm.tile, true);   // every tile sorted
      for (int kk = 2 * kLongSmem; kk <= N; kk <<= 1) {
        for (int m = kk >> 1; m >= kLongSmem; m >>= 1) {     // the long-distance steps, in global memory
          for (int t = threadIdx.x; t < N / 2; t += blockDim.x) {
            const int lo_bits = t & (m - 1);
            const int i = ((t - lo_bits) << 1) | lo_bits;
            const int j = m == (kk >> 1) ? (i ^ (kk - 1)) : (i | m);
            if (j < n) {
              const uint32_t x = g[i], y = g[j];
              if (x > y) {
                g[i] = y;
                g[j] = x;
              }
            }
          }
          __syncthreads();
        }
        bitonic_tiles_local(g, n, sm.tile, false);   // this merge's half-cleaners below the tile size
      }
    }
    __syncthreads();
  }
}

// per chunk: [item begin, item end) of the sorted items, the destination group, and where the
// chunk's sum goes (-1: straight into dM, else its partial slot) — one 16-byte load in pass 1
struct ChunkInfo {
  int32_t begin, end;
  uint32_t group;
  int32_t dst;
};

__global__ void emb_chunkmap_kernel(const int32_t* __restrict__ start, const int32_t* __restrict__ cnt,
                                    int64_t ngroups, const int32_t* __restrict__ choff,
                                    const int32_t* __restrict__ loff, ChunkInfo* __restrict__ info,
                                    int32_t* __restrict__ long_n, int32_t* __restrict__ long_list) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  const int32_t h = start[g];
  const int32_t e = h + cnt[g];
  const int c = (e - h + kW - 1) / kW;
  if (c > 1) long_list[atomicAdd(long_n, 1)] = int32_t(g);   // pass 2 visits only these (any order)
  for (int k = 0; k < c; ++k) {   // a Zipf-hot group writes its few dozen entries serially
    ChunkInfo ci;
    ci.begin = h + k * kW;
    ci.end = min(e, ci.begin + kW);
    ci.group = uint32_t(g);
    ci.dst = c == 1 ? -1 : loff[g] + k;
    info[choff[g] + k] = ci;
  }
}

// sum of one chunk's terms in item order.  The chunk is warp-uniform; lane k decodes item
// it0 + k once (index arithmetic, sign, lambda) and the warp broadcasts it with shuffles, so
// the integer work is per item instead of per item and lane; 8 dOut loads in flight.
__device__ __forceinline__ float chunk_sum(const ChunkInfo& ci, const uint32_t* __restrict__ vals,
                                           const float* __restrict__ dOut, int dim, int chunk, int q, int G, int A,
                                           const DetLam& L, int lane) {
  float acc = 0.f;
  constexpr int U = 8;
  for (int it0 = ci.begin; it0 < ci.end; it0 += 32) {
    int myb = 0, mycb = dim;   // row, first column of the item's A slots (dim = contributes nothing)
    float mys = 0.f;           // g * lambda
    if (it0 + lane < ci.end) {
      const uint32_t v = __ldg(vals + it0 + lane);
      const int item = int(v >> 1);   // < 2^30: 32-bit index arithmetic
      const int p = item / G;
      const int i = item - p * G;
      myb = p / q;
      mycb = (p - myb * q) * chunk + i * A;
      const float lam = L.lam[myb / L.n];
      mys = (v & 1u) ? -lam : lam;
    }
    const int cnt = min(32, ci.end - it0);
    for (int k0 = 0; k0 < cnt; k0 += U) {
      float t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u;   // k < 32 always; items past cnt carry mycb = dim
        const int b = __shfl_sync(0xffffffffu, myb, k);
        const int col = __shfl_sync(0xffffffffu, mycb, k) + lane;
        const float sl = __shfl_sync(0xffffffffu, mys, k);
        t[u] = 0.f;
        if (k < cnt && lane < A && col < dim)   // padded tail of the last chunk (R16): nothing
          t[u] = sl * __ldg(dOut + int64_t(b) * dim + col);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += t[u];
    }
  }
  return acc;
}

// pass 1: one warp per chunk, two chunks in flight per warp; lanes 0..A-1 own the group's A
// slots.  A single-chunk group goes straight to dM; a longer one leaves a partial.
__global__ void emb_chunk_kernel(float* __restrict__ dM, float* __restrict__ partial,
                                 const uint32_t* __restrict__ vals, const ChunkInfo* __restrict__ info,
                                 int64_t nseg, const int32_t* __restrict__ nch,
                                 const int32_t* __restrict__ choff, const float* __restrict__ dOut, int dim, int chunk,
                                 int q, int G, int A, const __grid_constant__ DetLam lam, int64_t mem_size) {
  const int lane = threadIdx.x & 31;
  if (nseg == 0) return;
  const int64_t total = int64_t(choff[nseg - 1]) + nch[nseg - 1];
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < total; c += 2 * nwarps) {
    const int64_t c2 = c + nwarps;
    const ChunkInfo i1 = info[c];
    ChunkInfo i2{0, 0, 0, -2};
    if (c2 < total) i2 = info[c2];
    const float s1 = chunk_sum(i1, vals, dOut, dim, chunk, q, G, A, lam, lane);
    const float s2 = chunk_sum(i2, vals, dOut, dim, chunk, q, G, A, lam, lane);
    if (lane >= A) continue;
    const ChunkInfo* ci[2] = {&i1, &i2};
    const float sum[2] = {s1, s2};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const ChunkInfo& x = *ci[u];
      if (x.dst == -2) continue;
      if (x.dst < 0) {
        const int64_t sl = int64_t(x.group) * A + lane;
        if (sl < mem_size) dM[sl] += sum[u];
      } else {
        partial[int64_t(x.dst) * A + lane] = sum[u];
      }
    }
  }
}

// pass 1, sub-warp version (A % 4 == 0, A <= 32): L = A / 4 lanes own one chunk (lane r of the
// sub-group holds slots 4r .. 4r + 3 of the group as a float4), so a warp works on 32 / L chunks
// at once (C4 at A = 32: 4, at A = 8: 16) instead of two — the pass is latency-bound (a few
// items per group, ~4 dependent round trips each), so more chunks in flight is what pays.  Each
// slot still adds its chunk's terms in item order (the same order as the warp version).
__global__ void __launch_bounds__(256, 8) emb_chunk_sub_kernel(float* __restrict__ dM, float* __restrict__ partial,
                                     const uint32_t* __restrict__ vals, const ChunkInfo* __restrict__ info,
                                     int64_t nseg, const int32_t* __restrict__ nch,
                                     const int32_t* __restrict__ choff, const float* __restrict__ dOut, int dim,
                                     int chunk, int q, int G, int A, const __grid_constant__ DetLam lam,
                                     int64_t mem_size) {
  const int L = A >> 2;                       // lanes per chunk
  const int r = (threadIdx.x & 31) % L;       // this lane's float4 of the group's A slots
  if (nseg == 0) return;
  const int64_t total = int64_t(choff[nseg - 1]) + nch[nseg - 1];
  const int64_t nsub = (int64_t(gridDim.x) * blockDim.x) / L;
  // the next chunk's descriptor is loaded an iteration ahead (one dependent round trip fewer per
  // chunk in this latency-bound pass: C4 0.628 -> 0.597 ms; also pre-loading its first item words
  // or 8 items per round of loads was slower); 8 resident blocks per SM (32 registers): 0.563 ms
  int64_t c = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  ChunkInfo nxt = c < total ? info[c] : ChunkInfo{0, 0, 0, -2};
  for (; c < total; c += nsub) {
    const ChunkInfo ci = nxt;
    if (c + nsub < total) nxt = info[c + nsub];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int it = ci.begin;
    constexpr int U = 4;
    for (; it + U <= ci.end; it += U) {      // U items' loads in flight, summed in item order
      float4 t[U];
      float sc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = __ldg(vals + it + u);
        const int item = int(v >> 1);
        const int p = item / G;
        const int i = item - p * G;
        const int b = p / q;
        const int col = (p - b * q) * chunk + i * A + 4 * r;
        const float l = lam.lam[b / lam.n];
        sc[u] = (v & 1u) ? -l : l;
        t[u] = col < dim ? __ldg(reinterpret_cast<const float4*>(dOut + int64_t(b) * dim + col))
                         : make_float4(0.f, 0.f, 0.f, 0.f);   // padded tail of the last chunk (R16)
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc.x += sc[u] * t[u].x;
        acc.y += sc[u] * t[u].y;
        acc.z += sc[u] * t[u].z;
        acc.w += sc[u] * t[u].w;
      }
    }
    for (; it < ci.end; ++it) {
      const uint32_t v = __ldg(vals + it);
      const int item = int(v >> 1);
      const int p = item / G;
      const int i = item - p * G;
      const int b = p / q;
      const int col = (p - b * q) * chunk + i * A + 4 * r;
      const float l = lam.lam[b / lam.n];
      const float sc = (v & 1u) ? -l : l;
      if (col < dim) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(dOut + int64_t(b) * dim + col));
        acc.x += sc * t.x;
        acc.y += sc * t.y;
        acc.z += sc * t.z;
        acc.w += sc * t.w;
      }
    }
    if (ci.dst < 0) {
      const int64_t sl = int64_t(ci.group) * A + 4 * r;
      if (sl + 4 <= mem_size) {
        float4* d = reinterpret_cast<float4*>(dM + sl);
        float4 o = *d;
        o.x += acc.x; o.y += acc.y; o.z += acc.z; o.w += acc.w;
        *d = o;
      } else {
        const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
        for (int k = 0; k < 4 && sl + k < mem_size; ++k) dM[sl + k] += a4[k];
      }
    } else {
      *reinterpret_cast<float4*>(partial + int64_t(ci.dst) * A + 4 * r) = acc;
    }
  }
}

// pass 2: one warp per multi-chunk group (the list emb_chunkmap_kernel appended; each group is
// summed on its own, so the list order does not matter): its partials in chunk order, then dM
__global__ void emb_longseg_kernel(float* __restrict__ dM, const float* __restrict__ partial,
                                   const int32_t* __restrict__ long_n, const int32_t* __restrict__ long_list,
                                   const int32_t* __restrict__ nch, const int32_t* __restrict__ loff, int A,
                                   int64_t mem_size) {
  const int lane = threadIdx.x & 31;
  const int64_t nlong = *long_n;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < nlong; j += nwarps) {
    const int64_t g = long_list[j];
    const int c = nch[g];
    if (lane >= A) continue;
    float acc = 0.f;
    for (int k = 0; k < c; ++k) acc += partial[(int64_t(loff[g]) + k) * A + lane];
    const int64_t s = g * A + lane;
    if (s < mem_size) dM[s] += acc;
  }
}

}  // namespace

namespace {
roast_status_t embed_bwd_det_group(Ctx* c, const Module* const* mods, int nt, const int64_t* idx, int64_t n,
                                   const float* dOut, cudaStream_t s);
}

roast_status_t embed_bwd_deterministic(Ctx* c, const Module* const* mods, int nt, const int64_t* idx, int64_t n,
                                       const float* dOut, cudaStream_t s) {
  // groups of kDetTables tables, one after the other (a fixed order across groups too)
  for (int t0 = 0; t0 < nt; t0 += kDetTables) {
    const int k = std::min(nt - t0, kDetTables);
    if (roast_status_t st = embed_bwd_det_group(c, mods + t0, k, idx + t0 * n, n,
                                                dOut + t0 * n * int64_t(mods[0]->dim), s))
      return st;
  }
  return ROAST_OK;
}

namespace {
roast_status_t embed_bwd_det_group(Ctx* c, const Module* const* mods, int nt, const int64_t* idx, int64_t n,
                                   const float* dOut, cudaStream_t s) {
  const Module& m = *mods[0];
  const int64_t np = int64_t(nt) * n * m.chunks_per_row;
  if (np == 0) return ROAST_OK;
  const int A = int(m.hash.align);
  const int G = m.chunk / A;
  const int64_t ni = np * G;
  for (int t = 1; t < nt; ++t)
    if (mods[t]->hash.align != m.hash.align || mods[t]->chunk != m.chunk || mods[t]->dim != m.dim)
      return fail(ROAST_ERR_CONFIG, "deterministic multi-table backward needs equal dim, chunk and alignment");
  const int64_t ng = c->mem_size / A + G;   // slot groups an item can land in
  if (ni >= (int64_t(1) << 30) || ng >= (int64_t(1) << 31) - 1 || A > 32)
    return fail(ROAST_ERR_UNSUPPORTED, "deterministic embedding backward: too many items or slot groups");
  DetTables T{};
  DetLam L{};
  for (int t = 0; t < nt; ++t) {
    T.h[t] = mods[t]->hash;
    T.rows[t] = mods[t]->rows;
    T.lam[t] = L.lam[t] = mods[t]->lam;
  }
  T.n = n;
  L.n = int(n);
  const int ng1 = int(ng) + 1;
  const int64_t max_segs = ni / (kSmall + 1) + 1;   // groups longer than kSmall, per size-class list
  const int64_t max_long = 2 * (ni / kW) + 2;       // chunks of multi-chunk groups (each has > kW items)
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                ng1, s);
  // [group | vals | sorted (ni u32 each) | rank (ni) | cnt | start | nch | choff | nlong | loff (ng + 1
  //  each) | seg begin / end (max_segs each) | info | partial | long list | scalars | temp]
  const int64_t ninfo = ng1 + ni / kW + 1;   // chunks <= groups + ni / kW
  const size_t bytes = size_t(ni) * 16 + size_t(ng1) * 24 + size_t(max_segs) * 24 + 32 + size_t(ninfo) * 16 +
                       size_t(max_long) * A * 4 + size_t(ni / kW + 2) * 4 + 1024 + temp;
  Scratch ws;
  roast_status_t st = scratch_alloc(ws, bytes, s);
  if (st) return st;
  uint8_t* base = ws.as<uint8_t>();
  uint32_t* grp = reinterpret_cast<uint32_t*>(base);
  uint32_t* vals = grp + ni;
  uint32_t* sorted = vals + ni;
  int32_t* rank = reinterpret_cast<int32_t*>(sorted + ni);
  int32_t* cnt = rank + ni;
  int32_t* start = cnt + ng1;
  int32_t* nch = start + ng1;
  int32_t* choff = nch + ng1;
  int32_t* nlong = choff + ng1;
  int32_t* loff = nlong + ng1;
  int32_t* seg_b = loff + ng1;           // 3 size classes x max_segs
  int32_t* seg_e = seg_b + 3 * max_segs;
  ChunkInfo* info = reinterpret_cast<ChunkInfo*>((reinterpret_cast<uintptr_t>(seg_e + 3 * max_segs) + 15) & ~uintptr_t(15));
  float* partial = reinterpret_cast<float*>(info + ninfo);
  int32_t* long_list = reinterpret_cast<int32_t*>(partial + max_long * A);
  int32_t* scal = reinterpret_cast<int32_t*>((reinterpret_cast<uintptr_t>(long_list + ni / kW + 2) + 15) & ~uintptr_t(15));
  int32_t* long_n = scal;
  int32_t* seg_n = scal + 1;   // 3 counters
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(scal + 4) + 255) & ~uintptr_t(255));
  ROAST_CUDA_CHECK(cudaMemsetAsync(cnt, 0, size_t(ng1) * sizeof(int32_t), s));
  ROAST_CUDA_CHECK(cudaMemsetAsync(scal, 0, 4 * sizeof(int32_t), s));
  emb_items_kernel<<<unsigned((np + 255) / 256), 256, 0, s>>>(T, idx, int64_t(nt) * n, m.chunks_per_row, G, grp, vals,
                                                              rank, cnt, c->d_err);
  ROAST_CUDA_CHECK(cudaGetLastError());
  size_t t1 = temp;
  ROAST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, t1, cnt, start, ng1, s));
  emb_place_kernel<<<unsigned((ni + 255) / 256), 256, 0, s>>>(grp, vals, rank, start, ni, sorted);
  ROAST_CUDA_CHECK(cudaGetLastError());
  emb_order_kernel<<<unsigned((ng + 255) / 256), 256, 0, s>>>(sorted, start, cnt, ng, nch, nlong, seg_n, seg_b, seg_e,
                                                              max_segs);
  ROAST_CUDA_CHECK(cudaGetLastError());
  emb_medsort_kernel<<<148 * 4, 256, 0, s>>>(sorted, seg_n, seg_b, seg_e);
  ROAST_CUDA_CHECK(cudaGetLastError());
  int end_bit = 1;   // item values are (item << 1) | sign < 2 ni
  while (end_bit < 32 && (int64_t(1) << end_bit) < 2 * ni) ++end_bit;
  emb_longsort_kernel<false><<<148 * 8, kLongThreads, 0, s>>>(sorted, seg_n + 1, seg_b + max_segs, seg_e + max_segs,
                                                             end_bit);
  ROAST_CUDA_CHECK(cudaGetLastError());
  emb_longsort_kernel<true><<<148, kLongThreads, 0, s>>>(sorted, seg_n + 2, seg_b + 2 * max_segs, seg_e + 2 * max_segs,
                                                       end_bit);
  ROAST_CUDA_CHECK(cudaGetLastError());
  t1 = temp;
  ROAST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, t1, nch, choff, ng1, s));
  t1 = temp;
  ROAST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, t1, nlong, loff, ng1, s));
  emb_chunkmap_kernel<<<unsigned((ng + 255) / 256), 256, 0, s>>>(start, cnt, ng, choff, loff, info, long_n, long_list);
  ROAST_CUDA_CHECK(cudaGetLastError());
  const int grid = 148 * 8;
  if (A % 4 == 0 && A <= 32 && !getenv("ROAST_EMB_DET_WARP"))
    emb_chunk_sub_kernel<<<148 * 16, 256, 0, s>>>(c->dM, partial, sorted, info, ng, nch, choff, dOut, m.dim, m.chunk,
                                                 m.chunks_per_row, G, A, L, c->mem_size);
  else
    emb_chunk_kernel<<<grid, 256, 0, s>>>(c->dM, partial, sorted, info, ng, nch, choff, dOut, m.dim, m.chunk,
                                          m.chunks_per_row, G, A, L, c->mem_size);
  ROAST_CUDA_CHECK(cudaGetLastError());
  emb_longseg_kernel<<<148 * 2, 256, 0, s>>>(c->dM, partial, long_n, long_list, nch, loff, A, c->mem_size);
  ROAST_CUDA_CHECK(cudaGetLastError());
  c->launches += 12;   // (+ two memsets)
  return ROAST_OK;
}
}  // namespace

}  // namespace roast
