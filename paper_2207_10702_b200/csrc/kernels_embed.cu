// kernels_embed.cu — ROAST/ROBE block embedding (the L operation, K6/K7).
//
//   out[b, jZ + o] = g(c) * fp32(lambda * M[h1(c) + o]),  c = idx[b] * ceil(d/Z) + j
//   (§4.1 "Lookup"; chunk numbering R16)
//   dM[h1(c) + o] += lambda * g(c) * dOut[b, jZ + o]      (duplicates add, R15)
//
// Mapping to the machine: a warp takes 32 (row, chunk) pairs at a time; lane p
// evaluates the hash of pair p once (offset + sign), then the warp streams the
// 32 chunks' bytes with 16-byte vector loads, looking each pair's offset up by
// shuffle.  Chunks are Z contiguous fp32 of M (the ROBE coalescing argument,
// P:247), at 32-byte-aligned offsets (A = 8).  Backward uses 16-byte vector
// atomics (red.global.add.v4.f32).
#include "roast_internal.h"

namespace roast {
namespace {

struct EmbArgs {
  ModuleHash hash;
  int64_t rows;
  int dim, chunk, q;  // q = chunks per row
  float lam;
};

__device__ __forceinline__ void pair_hash(const EmbArgs& a, const int64_t* idx, int64_t n, int64_t p,
                                          int64_t& off, float& sg, int64_t& b, int& j, int32_t* err) {
  off = -1;
  sg = 0.f;
  b = p / a.q;
  j = int(p - b * a.q);
  if (b >= n) return;
  int64_t r = idx[b];
  if (r < 0 || r >= a.rows) {
    atomicOr(err, 1);
    return;  // out of range -> zero row, sticky BOUNDS
  }
  uint64_t key = uint64_t(r) * uint64_t(a.q) + uint64_t(j);
  off = int64_t(a.hash.offset(key));
  sg = float(a.hash.sign(key));
}

template <bool kBwd, int U>
__global__ void __launch_bounds__(256) embed_kernel(EmbArgs a, const int64_t* __restrict__ idx, int64_t n,
                                                    const float* __restrict__ M, float* __restrict__ out,
                                                    const float* __restrict__ dOut, float* __restrict__ dM,
                                                    int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t npairs = n * a.q;
  const int v_per_chunk = a.chunk >> 2;  // float4 per chunk
  for (int64_t base = warp * 32; base < npairs; base += nwarps * 32) {
    int64_t off, b;
    float sg;
    int j;
    pair_hash(a, idx, n, base + lane, off, sg, b, j, err);
    // 32 pairs x Z/4 float4 per pair; each lane moves 8 float4 per batch with all 8
    // loads in flight before the first use (memory-level parallelism for the gathers)
    const int total = 32 * v_per_chunk;
    for (int e0 = 0; e0 < total; e0 += 32 * U) {
      float4 val[U];
      int64_t dst[U];
      float scl[U];
      int st[U];  // 0: skip, 1: write (zeros if invalid row), 2: data
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * 32 + lane;
        const int pp = e / v_per_chunk;
        const int part = e - pp * v_per_chunk;
        const int64_t poff = __shfl_sync(0xffffffff, off, pp & 31);
        const float psg = __shfl_sync(0xffffffff, sg, pp & 31);
        const int64_t pb = __shfl_sync(0xffffffff, b, pp & 31);
        const int pj = __shfl_sync(0xffffffff, j, pp & 31);
        const int col = pj * a.chunk + part * 4;
        st[u] = (e < total && pb < n && col < a.dim) ? (poff >= 0 ? 2 : 1) : 0;   // R16 padded tail
        scl[u] = kBwd ? psg * a.lam : psg;
        dst[u] = kBwd ? poff + part * 4 : pb * a.dim + col;
        val[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (st[u] == 2)
          val[u] = __ldg(reinterpret_cast<const float4*>(kBwd ? dOut + pb * a.dim + col : M + poff + part * 4));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!kBwd) {
          if (st[u] == 0) continue;
          // g * fp32(lambda * M): one rounding, then an exact sign flip
          const float4 m = val[u];
          const float4 v = make_float4(scl[u] * __fmul_rn(a.lam, m.x), scl[u] * __fmul_rn(a.lam, m.y),
                                       scl[u] * __fmul_rn(a.lam, m.z), scl[u] * __fmul_rn(a.lam, m.w));
          *reinterpret_cast<float4*>(out + dst[u]) = v;
        } else {
          if (st[u] != 2) continue;
          const float4 g = val[u];
          atomicAdd(reinterpret_cast<float4*>(dM + dst[u]),
                    make_float4(scl[u] * g.x, scl[u] * g.y, scl[u] * g.z, scl[u] * g.w));
        }
      }
    }
  }
}

__global__ void chunk_map_kernel(EmbArgs a, const int64_t* __restrict__ rows, int64_t n, int64_t* __restrict__ off,
                                 int8_t* __restrict__ sgn) {
  int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n * a.q) return;
  int64_t b = p / a.q;
  int j = int(p - b * a.q);
  uint64_t key = uint64_t(rows[b]) * uint64_t(a.q) + uint64_t(j);
  off[p] = int64_t(a.hash.offset(key));
  sgn[p] = int8_t(a.hash.sign(key));
}

EmbArgs emb_args(const Module& m) {
  EmbArgs a;
  a.hash = m.hash;
  a.rows = m.rows;
  a.dim = m.dim;
  a.chunk = m.chunk;
  a.q = m.chunks_per_row;
  a.lam = m.lam;
  return a;
}

int emb_grid(int64_t n, int q) {
  int64_t warps = (n * q + 31) / 32;
  int64_t blocks = (warps + 7) / 8;
  int64_t cap = 148 * 8;  // persistent-ish: up to 8 CTAs of 8 warps per SM
  if (blocks > cap) blocks = cap;
  return int(blocks < 1 ? 1 : blocks);
}

}  // namespace

cudaError_t launch_embed_fwd(const Ctx* c, const Module& m, const int64_t* idx, int64_t n, float* out,
                             cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  static const int U = getenv("ROAST_EMB_U") ? atoi(getenv("ROAST_EMB_U")) : 4;
  if (U == 8) embed_kernel<false, 8><<<emb_grid(n, m.chunks_per_row), 256, 0, s>>>(emb_args(m), idx, n, c->M, out, nullptr, nullptr, c->d_err);
  else embed_kernel<false, 4><<<emb_grid(n, m.chunks_per_row), 256, 0, s>>>(emb_args(m), idx, n, c->M, out, nullptr,
                                                                      nullptr, c->d_err);
  return cudaGetLastError();
}

cudaError_t launch_embed_bwd(const Ctx* c, const Module& m, const int64_t* idx, int64_t n, const float* dOut,
                             cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  static const int U = getenv("ROAST_EMB_U") ? atoi(getenv("ROAST_EMB_U")) : 4;
  if (U == 8) embed_kernel<true, 8><<<emb_grid(n, m.chunks_per_row), 256, 0, s>>>(emb_args(m), idx, n, nullptr, nullptr, dOut, c->dM, c->d_err);
  else embed_kernel<true, 4><<<emb_grid(n, m.chunks_per_row), 256, 0, s>>>(emb_args(m), idx, n, nullptr, nullptr, dOut,
                                                                     c->dM, c->d_err);
  return cudaGetLastError();
}

cudaError_t launch_chunk_map(const Ctx* c, const Module& m, const int64_t* rows, int64_t n, int64_t* off,
                             int8_t* sgn, cudaStream_t s) {
  (void)c;
  int64_t tot = n * m.chunks_per_row;
  if (tot == 0) return cudaSuccess;
  chunk_map_kernel<<<unsigned((tot + 255) / 256), 256, 0, s>>>(emb_args(m), rows, n, off, sgn);
  return cudaGetLastError();
}

}  // namespace roast
