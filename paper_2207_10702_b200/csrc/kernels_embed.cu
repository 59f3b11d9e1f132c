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
  int stream_hint;  // 1: evict-first hints on the streamed operands (out / dOut, idx)
};

// kT tables of equal dim / chunk in one launch (roast_embedding_{fwd,bwd}_multi): the
// batch is the table-major concatenation, row g in [0, kT n) belongs to table g / n.
template <int kT>
struct EmbBatch {
  EmbArgs t[kT];
  int ntables;
  int64_t n_per_table;
};

__device__ __forceinline__ int64_t load_row(const EmbArgs& a, const int64_t* idx, int64_t n, int64_t p) {
  const int64_t b = p / a.q;
  if (b >= n) return -1;
  return a.stream_hint ? __ldcs(idx + b) : __ldg(idx + b);
}

// pair p = (row g, chunk j) of the concatenated batch -> offset, sign * lambda-free sign, row, chunk, lambda
template <int kT>
__device__ __forceinline__ void pair_hash(const EmbBatch<kT>& B, int64_t r, int64_t n, int64_t p, int64_t& off,
                                          float& sg, float& lam, int64_t& g, int& j, int32_t* err) {
  const EmbArgs& a0 = B.t[0];
  off = -1;
  sg = 0.f;
  lam = 0.f;
  g = p / a0.q;
  j = int(p - g * a0.q);
  if (g >= n) return;
  const int t = kT == 1 ? 0 : int(g / B.n_per_table);
  const EmbArgs& a = B.t[t];
  lam = a.lam;
  if (r < 0 || r >= a.rows) {
    atomicOr(err, 1);
    return;  // out of range -> zero row, sticky BOUNDS
  }
  uint64_t key = uint64_t(r) * uint64_t(a.q) + uint64_t(j);
  off = int64_t(a.hash.offset(key));
  sg = float(a.hash.sign(key));
}

#ifndef ROAST_EMB_MINB
#define ROAST_EMB_MINB 4
#endif
// n = total rows of the (concatenated) batch; out / dOut are n x dim
template <bool kBwd, int kT, int U>
__global__ void __launch_bounds__(256, ROAST_EMB_MINB) embed_kernel(const __grid_constant__ EmbBatch<kT> B,
                                                                    const int64_t* __restrict__ idx, int64_t n,
                                                                    const float* __restrict__ M,
                                                                    float* __restrict__ out,
                                                                    const float* __restrict__ dOut,
                                                                    float* __restrict__ dM, int32_t* err) {
  const EmbArgs& a = B.t[0];  // dim / chunk / q / hint are common to all tables
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t npairs = n * a.q;
  const int v_per_chunk = a.chunk >> 2;  // float4 per chunk
  // the next iteration's row id is loaded before this iteration's gathers, hiding the
  // dependent idx -> hash -> M latency chain behind one iteration of work
  int64_t r_next = warp * 32 < npairs ? load_row(a, idx, n, warp * 32 + lane) : -1;
  for (int64_t base = warp * 32; base < npairs; base += nwarps * 32) {
    int64_t off, g;
    float sg, lam;
    int j;
    const int64_t r = r_next;
    if (base + nwarps * 32 < npairs) r_next = load_row(a, idx, n, base + nwarps * 32 + lane);
    pair_hash(B, r, n, base + lane, off, sg, lam, g, j, err);
    // 32 pairs x Z/4 float4 per pair; each lane moves U float4 per batch with all U
    // loads in flight before the first use (memory-level parallelism for the gathers)
    const int total = 32 * v_per_chunk;
    for (int e0 = 0; e0 < total; e0 += 32 * U) {
      float4 val[U];
      int64_t dst[U];
      float scl[U], lm[U];
      int st[U];  // 0: skip, 1: write (zeros if invalid row), 2: data
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * 32 + lane;
        const int pp = e / v_per_chunk;
        const int part = e - pp * v_per_chunk;
        const int64_t poff = __shfl_sync(0xffffffff, off, pp & 31);
        const float psg = __shfl_sync(0xffffffff, sg, pp & 31);
        const int64_t pg = __shfl_sync(0xffffffff, g, pp & 31);
        const int pj = __shfl_sync(0xffffffff, j, pp & 31);
        lm[u] = kT == 1 ? a.lam : __shfl_sync(0xffffffff, lam, pp & 31);
        const int col = pj * a.chunk + part * 4;
        st[u] = (e < total && pg < n && col < a.dim) ? (poff >= 0 ? 2 : 1) : 0;   // R16 padded tail
        scl[u] = kBwd ? psg * lm[u] : psg;
        dst[u] = kBwd ? poff + part * 4 : pg * a.dim + col;
        val[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (st[u] == 2) {
          if (kBwd)
            val[u] = a.stream_hint ? __ldcs(reinterpret_cast<const float4*>(dOut + pg * a.dim + col))
                                   : __ldg(reinterpret_cast<const float4*>(dOut + pg * a.dim + col));
          else
            val[u] = __ldg(reinterpret_cast<const float4*>(M + poff + part * 4));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!kBwd) {
          if (st[u] == 0) continue;
          // g * fp32(lambda * M): one rounding, then an exact sign flip
          const float4 m = val[u];
          const float4 v = make_float4(scl[u] * __fmul_rn(lm[u], m.x), scl[u] * __fmul_rn(lm[u], m.y),
                                       scl[u] * __fmul_rn(lm[u], m.z), scl[u] * __fmul_rn(lm[u], m.w));
          if (a.stream_hint) __stcs(reinterpret_cast<float4*>(out + dst[u]), v);
          else *reinterpret_cast<float4*>(out + dst[u]) = v;
        } else {
          if (st[u] != 2) continue;
          const float4 gv = val[u];
          atomicAdd(reinterpret_cast<float4*>(dM + dst[u]),
                    make_float4(scl[u] * gv.x, scl[u] * gv.y, scl[u] * gv.z, scl[u] * gv.w));
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
  static const int hint = getenv("ROAST_EMB_CS") ? atoi(getenv("ROAST_EMB_CS")) : 0;
  a.stream_hint = hint;
  return a;
}

template <bool kBwd, int kT>
int emb_grid(int64_t n, int q) {
  int64_t warps = (n * q + 31) / 32;
  int64_t blocks = (warps + 7) / 8;
  // persistent: exactly the CTAs that are co-resident on all SMs (no second partial wave)
  static const int64_t cap = [] {
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, embed_kernel<kBwd, kT, 4>, 256, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return int64_t(per_sm < 1 ? 1 : per_sm) * int64_t(sms < 1 ? 148 : sms);
  }();
  if (blocks > cap) blocks = cap;
  return int(blocks < 1 ? 1 : blocks);
}

template <bool kBwd, int kT>
cudaError_t launch_embed(const Ctx* c, const Module* const* mods, int nt, const int64_t* idx, int64_t n,
                         float* out, const float* dOut, cudaStream_t s) {
  EmbBatch<kT> B;
  for (int t = 0; t < nt; ++t) B.t[t] = emb_args(*mods[t]);
  for (int t = nt; t < kT; ++t) B.t[t] = B.t[0];
  B.ntables = nt;
  B.n_per_table = n;
  const int64_t rows = n * nt;
  embed_kernel<kBwd, kT, 4><<<emb_grid<kBwd, kT>(rows, mods[0]->chunks_per_row), 256, 0, s>>>(
      B, idx, rows, c->M, out, dOut, c->dM, c->d_err);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_embed_fwd(const Ctx* c, const Module& m, const int64_t* idx, int64_t n, float* out,
                             cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const Module* mods[1] = {&m};
  return launch_embed<false, 1>(c, mods, 1, idx, n, out, nullptr, s);
}

cudaError_t launch_embed_bwd(const Ctx* c, const Module& m, const int64_t* idx, int64_t n, const float* dOut,
                             cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const Module* mods[1] = {&m};
  return launch_embed<true, 1>(c, mods, 1, idx, n, nullptr, dOut, s);
}

cudaError_t launch_embed_multi(const Ctx* c, const Module* const* mods, int nt, const int64_t* idx, int64_t n,
                               float* out, const float* dOut, cudaStream_t s) {
  if (n == 0 || nt == 0) return cudaSuccess;
  if (nt == 1) return dOut ? launch_embed<true, 1>(c, mods, 1, idx, n, nullptr, dOut, s)
                           : launch_embed<false, 1>(c, mods, 1, idx, n, out, nullptr, s);
  return dOut ? launch_embed<true, kEmbMaxTables>(c, mods, nt, idx, n, nullptr, dOut, s)
              : launch_embed<false, kEmbMaxTables>(c, mods, nt, idx, n, out, nullptr, s);
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
