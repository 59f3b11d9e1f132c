// kernels_embed_det.cu — deterministic embedding backward (a5, deterministic mode).
//
//   dM[h1(c) + o] += lambda * g(c) * dOut[b, jZ + o]     (R15, R19)
//
// The fast path scatters with vector atomics (order unspecified).  Here every slot is
// owned by one thread and summed in a fixed order:
//   1. key each (lookup b, chunk j) pair by its offset / A (the hash, on the device);
//   2. stable radix sort (CUB) -> pairs ordered by (offset, pair index);
//   3. for each 4-slot vector s, binary-search the pairs whose chunk [off, off + Z) covers s
//      (offsets in (s - Z, s]) and add their contributions in that order.
// Bitwise reproducible run to run; the same structure as the linear-layer K5 reduce.
#include <cub/device/device_radix_sort.cuh>

#include "roast_internal.h"

namespace roast {
namespace {

__global__ void emb_keys_kernel(ModuleHash h, const int64_t* __restrict__ idx, int64_t n, int64_t rows, int q,
                                uint32_t* __restrict__ keys, int32_t* __restrict__ vals, int32_t* err) {
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n * q) return;
  const int64_t b = p / q;
  const int j = int(p - b * q);
  const int64_t r = idx[b];
  if (r < 0 || r >= rows) {
    atomicOr(err, 1);
    keys[p] = 0xFFFFFFFFu;   // sorts last; the reduce never reaches it (no slot >= 2^32 * A)
    vals[p] = -1;
    return;
  }
  const uint64_t key = uint64_t(r) * uint64_t(q) + uint64_t(j);
  keys[p] = uint32_t(h.offset(key) / h.align);
  vals[p] = int32_t(p) | (h.sign(key) < 0 ? int32_t(0x80000000) : 0);   // sign in the top bit
}

__global__ void emb_det_reduce_kernel(float* __restrict__ dM, const uint32_t* __restrict__ keys,
                                      const int32_t* __restrict__ vals, int64_t npairs, const float* __restrict__ dOut,
                                      int dim, int chunk, int q, int align, float lam, int64_t mem_size) {
  const int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (s >= mem_size) return;
  // covering chunks: off in (s - Z, s]  <=>  key = off / A in [ceil((s - Z + 1) / A), floor(s / A)]
  const int64_t klo = s - chunk + 1 <= 0 ? 0 : (s - chunk + 1 + align - 1) / align;
  const int64_t khi = s / align;
  int64_t a = 0, e = npairs;
  while (a < e) {
    const int64_t mid = (a + e) >> 1;
    if (int64_t(keys[mid]) < klo) a = mid + 1; else e = mid;
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool any = false;
  for (int64_t i = a; i < npairs && int64_t(keys[i]) <= khi; ++i) {
    const int32_t v = vals[i];
    const int64_t p = int64_t(v & 0x7FFFFFFF);
    const float sc = (v < 0 ? -lam : lam);
    const int64_t b = p / q;
    const int j = int(p - b * q);
    const int o = int(s - int64_t(keys[i]) * align);      // position of s inside the chunk
    const int col = j * chunk + o;
    if (col >= dim) continue;                             // padded tail of the last chunk (R16)
    const float4 g = __ldg(reinterpret_cast<const float4*>(dOut + b * dim + col));
    acc.x += sc * g.x;
    acc.y += sc * g.y;
    acc.z += sc * g.z;
    acc.w += sc * g.w;
    any = true;
  }
  if (!any) return;
  float4* d = reinterpret_cast<float4*>(dM + s);
  float4 m = *d;
  m.x += acc.x;
  m.y += acc.y;
  m.z += acc.z;
  m.w += acc.w;
  *d = m;
}

}  // namespace

roast_status_t embed_bwd_deterministic(Ctx* c, const Module& m, const int64_t* idx, int64_t n, const float* dOut,
                                       cudaStream_t s) {
  const int64_t np = n * m.chunks_per_row;
  if (np == 0) return ROAST_OK;
  if (np >= (int64_t(1) << 31) || c->mem_size / m.hash.align >= (int64_t(1) << 32) - 1)
    return fail(ROAST_ERR_UNSUPPORTED, "deterministic embedding backward: too many pairs or slots");
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), int(np), 0,
                                  32, s);
  const size_t bytes = size_t(np) * 16 + temp + 256;
  roast_status_t st = ensure_ws(c, bytes, s);
  if (st) return st;
  uint8_t* base = reinterpret_cast<uint8_t*>(c->ws);
  uint32_t* k_in = reinterpret_cast<uint32_t*>(base);
  uint32_t* k_out = k_in + np;
  int32_t* v_in = reinterpret_cast<int32_t*>(k_out + np);
  int32_t* v_out = v_in + np;
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(v_out + np) + 255) & ~uintptr_t(255));
  emb_keys_kernel<<<unsigned((np + 255) / 256), 256, 0, s>>>(m.hash, idx, n, m.rows, m.chunks_per_row, k_in, v_in,
                                                             c->d_err);
  ROAST_CUDA_CHECK(cudaGetLastError());
  // invalid rows carry key 0xFFFFFFFF: sort all 32 bits when any could be present
  ROAST_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, temp, k_in, k_out, v_in, v_out, int(np), 0, 32, s));
  const int64_t vecs = (c->mem_size + 3) / 4;
  emb_det_reduce_kernel<<<unsigned((vecs + 255) / 256), 256, 0, s>>>(c->dM, k_out, v_out, np, dOut, m.dim, m.chunk,
                                                                      m.chunks_per_row, int(m.hash.align), m.lam,
                                                                      c->mem_size);
  ROAST_CUDA_CHECK(cudaGetLastError());
  c->launches += 3;
  return ROAST_OK;
}

}  // namespace roast
