// kernels_embed_det.cu — deterministic embedding backward (a5, deterministic mode).
//
//   dM[h1(c) + o] += lambda * g(c) * dOut[b, jZ + o]     (R15, R19)
//
// The fast path scatters with vector atomics (order unspecified).  Here every slot is summed
// in a fixed order, and only the slots some lookup touches are visited:
//   1. each (lookup b, chunk j) pair covers G = Z / A slot groups of A slots (offsets are
//      multiples of A); emit one item per (pair, group i) with the sort key
//      (offset / A + i) * G + (G - 1 - i)   — group first, then ascending chunk offset;
//   2. stable radix sort (CUB) -> items ordered by (group, chunk offset, pair index);
//   3. a group (a run of equal key / G) is cut into fixed chunks of 64 items; one warp per
//      chunk (lanes 0..A-1 own the group's A slots) adds the chunk's lambda * g * dOut terms
//      in item order; one-chunk groups add straight into dM, longer ones (Zipf-hot rows:
//      thousands of duplicates) leave partials that a second pass adds in chunk order.
// Bitwise reproducible run to run (every order is fixed by the sorted data, not by timing).
// Work is O(lookups), not O(|M|), and hot rows are summed in parallel.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

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

__global__ void emb_items_kernel(const __grid_constant__ DetTables T, const int64_t* __restrict__ idx, int64_t nlook, int q, int G,
                                 uint32_t* __restrict__ keys, int32_t* __restrict__ vals, int32_t* err,
                                 int32_t* __restrict__ nvalid) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p == 0) *nvalid = int32_t(nlook * q * G);   // lowered by emb_heads_kernel if rows were out of range
  if (p >= nlook * q) return;
  const int64_t b = p / q;
  const int j = int(p - b * q);
  const int t = int(b / T.n);
  const int64_t r = idx[b];
  if (r < 0 || r >= T.rows[t]) {
    atomicOr(err, 1);
    for (int i = 0; i < G; ++i) {   // sorts last; the reduce skips the sentinel group
      keys[p * G + i] = 0xFFFFFFFFu;
      vals[p * G + i] = -1;
    }
    return;
  }
  const uint64_t key = uint64_t(r) * uint64_t(q) + uint64_t(j);
  const uint32_t k0 = uint32_t(T.h[t].offset(key) / T.h[t].align);
  const int32_t neg = T.h[t].sign(key) < 0 ? int32_t(0x80000000) : 0;
  for (int i = 0; i < G; ++i) {
    keys[p * G + i] = (k0 + uint32_t(i)) * uint32_t(G) + uint32_t(G - 1 - i);
    vals[p * G + i] = int32_t(p * G + i) | neg;   // item index, sign in the top bit
  }
}

struct DetLam {   // lambda of each table and lookups per table (pass 1)
  float lam[kDetTables];
  int n;
};

__global__ void emb_heads_kernel(const uint32_t* __restrict__ keys, int64_t nitems, int G, uint8_t* __restrict__ head,
                                 int32_t* __restrict__ nvalid) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nitems) return;
  const uint32_t k = keys[i];
  const bool sent = k == 0xFFFFFFFFu;
  head[i] = !sent && (i == 0 || keys[i - 1] / uint32_t(G) != k / uint32_t(G));
  if (sent && (i == 0 || keys[i - 1] != 0xFFFFFFFFu)) *nvalid = int32_t(i);   // first sentinel
}

constexpr int kW = 64;   // items per chunk of a group's sum (fixed: the order is data-independent)

// per segment (group): number of kW-item chunks, and the same count for multi-chunk segments only
__global__ void emb_seginfo_kernel(const int32_t* __restrict__ heads, const int32_t* __restrict__ nseg_p,
                                   const int32_t* __restrict__ nvalid_p, int64_t nitems, int32_t* __restrict__ nch,
                                   int32_t* __restrict__ nlong) {
  const int64_t sg = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (sg > nitems) return;
  const int64_t nseg = *nseg_p;
  int32_t c = 0;
  if (sg < nseg) {
    const int64_t e = sg + 1 < nseg ? int64_t(heads[sg + 1]) : int64_t(*nvalid_p);
    c = int32_t((e - heads[sg] + kW - 1) / kW);
  }
  nch[sg] = c;
  nlong[sg] = c > 1 ? c : 0;
}

// per chunk: [item begin, item end) of the sorted items, the destination group, and where the
// chunk's sum goes (-1: straight into dM, else its partial slot) — one 16-byte load in pass 1
struct ChunkInfo {
  int32_t begin, end;
  uint32_t group;
  int32_t dst;
};

__global__ void emb_chunkmap_kernel(const uint32_t* __restrict__ keys, const int32_t* __restrict__ heads,
                                    const int32_t* __restrict__ nseg_p, const int32_t* __restrict__ nvalid_p,
                                    const int32_t* __restrict__ nch, const int32_t* __restrict__ choff,
                                    const int32_t* __restrict__ loff, int G, ChunkInfo* __restrict__ info,
                                    int32_t* __restrict__ long_n, int32_t* __restrict__ long_list) {
  const int64_t sg = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nseg = *nseg_p;
  if (sg >= nseg) return;
  const int32_t h = heads[sg];
  const int32_t e = sg + 1 < nseg ? heads[sg + 1] : *nvalid_p;
  const uint32_t group = keys[h] / uint32_t(G);
  const int c = nch[sg];
  if (c > 1) long_list[atomicAdd(long_n, 1)] = int32_t(sg);   // pass 2 visits only these (any order)
  for (int k = 0; k < c; ++k) {   // a Zipf-hot group writes its few dozen entries serially
    ChunkInfo ci;
    ci.begin = h + k * kW;
    ci.end = min(e, ci.begin + kW);
    ci.group = group;
    ci.dst = c == 1 ? -1 : loff[sg] + k;
    info[choff[sg] + k] = ci;
  }
}

// sum of one chunk's terms in item order.  The chunk is warp-uniform; lane k decodes item
// it0 + k once (index arithmetic, sign, lambda) and the warp broadcasts it with shuffles, so
// the integer work is per item instead of per item and lane; 8 dOut loads in flight.
__device__ __forceinline__ float chunk_sum(const ChunkInfo& ci, const int32_t* __restrict__ vals,
                                           const float* __restrict__ dOut, int dim, int chunk, int q, int G, int A,
                                           const DetLam& L, int lane) {
  float acc = 0.f;
  constexpr int U = 8;
  for (int it0 = ci.begin; it0 < ci.end; it0 += 32) {
    int myb = 0, mycb = dim;   // row, first column of the item's A slots (dim = contributes nothing)
    float mys = 0.f;           // g * lambda
    if (it0 + lane < ci.end) {
      const int32_t v = __ldg(vals + it0 + lane);
      const int item = v & 0x7FFFFFFF;   // < 2^30: 32-bit index arithmetic
      const int p = item / G;
      const int i = item - p * G;
      myb = p / q;
      mycb = (p - myb * q) * chunk + i * A;
      const float lam = L.lam[myb / L.n];
      mys = v < 0 ? -lam : lam;
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
                                 const int32_t* __restrict__ vals, const ChunkInfo* __restrict__ info,
                                 const int32_t* __restrict__ nseg_p, const int32_t* __restrict__ nch,
                                 const int32_t* __restrict__ choff, const float* __restrict__ dOut, int dim, int chunk,
                                 int q, int G, int A, const __grid_constant__ DetLam lam, int64_t mem_size) {
  const int lane = threadIdx.x & 31;
  const int64_t nseg = *nseg_p;
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
__global__ void emb_chunk_sub_kernel(float* __restrict__ dM, float* __restrict__ partial,
                                     const int32_t* __restrict__ vals, const ChunkInfo* __restrict__ info,
                                     const int32_t* __restrict__ nseg_p, const int32_t* __restrict__ nch,
                                     const int32_t* __restrict__ choff, const float* __restrict__ dOut, int dim,
                                     int chunk, int q, int G, int A, const __grid_constant__ DetLam lam,
                                     int64_t mem_size) {
  const int L = A >> 2;                       // lanes per chunk
  const int r = (threadIdx.x & 31) % L;       // this lane's float4 of the group's A slots
  const int64_t nseg = *nseg_p;
  if (nseg == 0) return;
  const int64_t total = int64_t(choff[nseg - 1]) + nch[nseg - 1];
  const int64_t nsub = (int64_t(gridDim.x) * blockDim.x) / L;
  for (int64_t c = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / L; c < total; c += nsub) {
    const ChunkInfo ci = info[c];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int it = ci.begin;
    constexpr int U = 4;
    for (; it + U <= ci.end; it += U) {      // U items' loads in flight, summed in item order
      float4 t[U];
      float sc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t v = __ldg(vals + it + u);
        const int item = v & 0x7FFFFFFF;
        const int p = item / G;
        const int i = item - p * G;
        const int b = p / q;
        const int col = (p - b * q) * chunk + i * A + 4 * r;
        const float l = lam.lam[b / lam.n];
        sc[u] = v < 0 ? -l : l;
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
      const int32_t v = __ldg(vals + it);
      const int item = v & 0x7FFFFFFF;
      const int p = item / G;
      const int i = item - p * G;
      const int b = p / q;
      const int col = (p - b * q) * chunk + i * A + 4 * r;
      const float l = lam.lam[b / lam.n];
      const float sc = v < 0 ? -l : l;
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
                                   const uint32_t* __restrict__ keys, const int32_t* __restrict__ heads,
                                   const int32_t* __restrict__ long_n, const int32_t* __restrict__ long_list,
                                   const int32_t* __restrict__ nch, const int32_t* __restrict__ loff, int G, int A,
                                   int64_t mem_size) {
  const int lane = threadIdx.x & 31;
  const int64_t nlong = *long_n;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < nlong; j += nwarps) {
    const int64_t sg = long_list[j];
    const int c = nch[sg];
    if (lane >= A) continue;
    float acc = 0.f;
    for (int k = 0; k < c; ++k) acc += partial[(int64_t(loff[sg]) + k) * A + lane];
    const int64_t s = int64_t(keys[heads[sg]] / uint32_t(G)) * A + lane;
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
  if (ni >= (int64_t(1) << 30) || (c->mem_size / A + G) * G >= (int64_t(1) << 32) - 1 || A > 32)
    return fail(ROAST_ERR_UNSUPPORTED, "deterministic embedding backward: too many items or slot groups");
  // sort only the key bits in use: keys < (|M| / A + G) * G
  int end_bit = 1;
  while (end_bit < 32 && (uint64_t(1) << end_bit) <= uint64_t((c->mem_size / A + G) * G)) ++end_bit;
  DetTables T{};
  DetLam L{};
  for (int t = 0; t < nt; ++t) {
    T.h[t] = mods[t]->hash;
    T.rows[t] = mods[t]->rows;
    T.lam[t] = L.lam[t] = mods[t]->lam;
  }
  T.n = n;
  L.n = int(n);
  const int ni1 = int(ni) + 1;
  size_t t_sort = 0, t_sel = 0, t_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t_sort, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), int(ni), 0, end_bit, s);
  cub::CountingInputIterator<int32_t> count_it(0);
  cub::DeviceSelect::Flagged(nullptr, t_sel, count_it, static_cast<const uint8_t*>(nullptr),
                             static_cast<int32_t*>(nullptr), static_cast<int32_t*>(nullptr), int(ni), s);
  cub::DeviceScan::ExclusiveSum(nullptr, t_scan, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                ni1, s);
  const size_t temp = std::max(t_sort, std::max(t_sel, t_scan));
  const int64_t max_long = 2 * (ni / kW) + 2;   // chunks of multi-chunk groups (each has > kW items)
  // [keys in | keys out | vals in | vals out | heads | nch | choff | nlong | loff (ni + 1 each) |
  //  partial (max_long x A fp32) | flags (u8) | 4 scalars | temp]
  const size_t bytes = size_t(ni) * 16 + size_t(ni1) * 20 + size_t(ni1 + ni / kW + 1) * 16 + 16 +
                       size_t(max_long) * A * 4 + size_t(ni) + 1024 + size_t(ni / kW + 2) * 4 + 16 + temp;
  Scratch ws;
  roast_status_t st = scratch_alloc(ws, bytes, s);
  if (st) return st;
  uint8_t* base = ws.as<uint8_t>();
  uint32_t* k_in = reinterpret_cast<uint32_t*>(base);
  uint32_t* k_out = k_in + ni;
  int32_t* v_in = reinterpret_cast<int32_t*>(k_out + ni);
  int32_t* v_out = v_in + ni;
  int32_t* heads = v_out + ni;
  int32_t* nch = heads + ni1;
  int32_t* choff = nch + ni1;
  int32_t* nlong = choff + ni1;
  int32_t* loff = nlong + ni1;
  ChunkInfo* info = reinterpret_cast<ChunkInfo*>((reinterpret_cast<uintptr_t>(loff + ni1) + 15) & ~uintptr_t(15));
  float* partial = reinterpret_cast<float*>(info + ni1 + ni / kW + 1);   // total chunks <= ni + ni / kW
  uint8_t* flags = reinterpret_cast<uint8_t*>(partial + max_long * A);
  int32_t* scal = reinterpret_cast<int32_t*>((reinterpret_cast<uintptr_t>(flags + ni) + 15) & ~uintptr_t(15));
  int32_t* nseg = scal;
  int32_t* nvalid = scal + 1;
  int32_t* long_n = scal + 2;
  int32_t* long_list = scal + 4;   // multi-chunk groups (each has > kW items): <= ni / kW of them
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(long_list + ni / kW + 2) + 255) & ~uintptr_t(255));
  ROAST_CUDA_CHECK(cudaMemsetAsync(long_n, 0, sizeof(int32_t), s));
  emb_items_kernel<<<unsigned((np + 255) / 256), 256, 0, s>>>(T, idx, int64_t(nt) * n, m.chunks_per_row, G, k_in,
                                                              v_in, c->d_err, nvalid);
  ROAST_CUDA_CHECK(cudaGetLastError());
  size_t t1 = temp;
  ROAST_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, t1, k_in, k_out, v_in, v_out, int(ni), 0, end_bit, s));
  emb_heads_kernel<<<unsigned((ni + 255) / 256), 256, 0, s>>>(k_out, ni, G, flags, nvalid);
  ROAST_CUDA_CHECK(cudaGetLastError());
  size_t t2 = temp;
  ROAST_CUDA_CHECK(cub::DeviceSelect::Flagged(tmp, t2, count_it, flags, heads, nseg, int(ni), s));
  emb_seginfo_kernel<<<unsigned((ni1 + 255) / 256), 256, 0, s>>>(heads, nseg, nvalid, ni, nch, nlong);
  ROAST_CUDA_CHECK(cudaGetLastError());
  size_t t3 = temp;
  ROAST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, t3, nch, choff, ni1, s));
  t3 = temp;
  ROAST_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp, t3, nlong, loff, ni1, s));
  emb_chunkmap_kernel<<<unsigned((ni1 + 255) / 256), 256, 0, s>>>(k_out, heads, nseg, nvalid, nch, choff, loff, G,
                                                                    info, long_n, long_list);
  ROAST_CUDA_CHECK(cudaGetLastError());
  const int grid = 148 * 8;
  if (A % 4 == 0 && A <= 32 && !getenv("ROAST_EMB_DET_WARP"))
    emb_chunk_sub_kernel<<<148 * 16, 256, 0, s>>>(c->dM, partial, v_out, info, nseg, nch, choff, dOut, m.dim,
                                                 m.chunk, m.chunks_per_row, G, A, L, c->mem_size);
  else
    emb_chunk_kernel<<<grid, 256, 0, s>>>(c->dM, partial, v_out, info, nseg, nch, choff, dOut, m.dim, m.chunk,
                                          m.chunks_per_row, G, A, L, c->mem_size);
  ROAST_CUDA_CHECK(cudaGetLastError());
  emb_longseg_kernel<<<148 * 2, 256, 0, s>>>(c->dM, partial, k_out, heads, long_n, long_list, nch, loff, G, A,
                                            c->mem_size);
  ROAST_CUDA_CHECK(cudaGetLastError());
  c->launches += 9;   // (+ one memset)
  return ROAST_OK;
}
}  // namespace

}  // namespace roast
