// kernels_ln.cu — LayerNorm of the ROASTed BERT workload: the
// N-operations stay plain, but at C3's 65 536 tokens torch's LayerNorm spends 0.85 ms
// per call (its parameter-gradient kernel alone 0.56 ms), more than the layer's ROAST GEMMs.
// Here one pass each way, memory-bound:
//   forward  : s = x (+ r, the residual, fused), mean / rstd per row, y = (s - mean) rstd g + b
//   backward : xhat = (s - mean) rstd, dxhat = dy g,
//              ds = rstd (dxhat - mean(dxhat) - xhat mean(dxhat xhat)),
//              dg = sum_rows dy xhat, db = sum_rows dy  (per-warp partials in registers, then a
//              fixed-order reduce: bitwise reproducible)
// One warp per row; lane l holds the 8-element vectors l, l + 32, ... of the row in registers;
// each warp keeps its next rows' loads in flight (forward: two rows at once, backward: the next
// row prefetched), which is what brings these HBM-bound passes near the copy bandwidth.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "roast_internal.h"

namespace roast {
namespace {

template <class T>
struct Vec8;
template <>
struct Vec8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* f) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 t = __bfloat1622float2(h[k]);
      f[2 * k] = t.x;
      f[2 * k + 1] = t.y;
    }
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float* f) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
  static __device__ __forceinline__ void round(float* f) {   // to the stored precision
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = __bfloat162float(__float2bfloat16_rn(f[k]));
  }
};
template <>
struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float* f) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(f[4], f[5], f[6], f[7]);
  }
  static __device__ __forceinline__ void round(float*) {}
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// The row data as loaded (raw) and widened to fp32 on use, so a warp can keep the next rows' loads
// in flight while it works on the current ones.
template <class T>
struct Raw8;
template <>
struct Raw8<__nv_bfloat16> {
  uint4 u;
  template <bool CS = false>   // CS: streaming (evict-first) load
  __device__ __forceinline__ void load(const __nv_bfloat16* p) {
    u = CS ? __ldcs(reinterpret_cast<const uint4*>(p)) : *reinterpret_cast<const uint4*>(p);
  }
  __device__ __forceinline__ void get(float* f) const {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 t = __bfloat1622float2(h[k]);
      f[2 * k] = t.x;
      f[2 * k + 1] = t.y;
    }
  }
};
template <>
struct Raw8<float> {
  float4 a, b;
  template <bool CS = false>
  __device__ __forceinline__ void load(const float* p) {
    a = CS ? __ldcs(reinterpret_cast<const float4*>(p)) : *reinterpret_cast<const float4*>(p);
    b = CS ? __ldcs(reinterpret_cast<const float4*>(p + 4)) : *reinterpret_cast<const float4*>(p + 4);
  }
  __device__ __forceinline__ void get(float* f) const {
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
};

// Forward: one warp per row, R rows of a warp in flight at once (their loads issued together).
template <class T, class P, int VPL, int R>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const T* __restrict__ x, const T* __restrict__ r,
                                                    const P* __restrict__ g, const P* __restrict__ b,
                                                    T* __restrict__ y, T* __restrict__ s_out,
                                                    float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                    int64_t rows, int n, float eps) {
  const int lane = threadIdx.x & 31;
  const int nv = n >> 3;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row0 = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * R; row0 < rows;
       row0 += nwarps * R) {
    Raw8<T> rx[R][VPL], rr[R][VPL];
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (row0 + q < rows && lane + 32 * k < nv) {
          const int64_t o = (row0 + q) * n + (lane + 32 * k) * 8;
          // two rows in flight = the large-row-count case, whose inputs are not L2-resident:
          // streaming loads leave L2 to the stores (65 536 x 768: 72 vs 114 us with plain loads)
          rx[q][k].template load<(R > 1)>(x + o);
          if (r) rr[q][k].template load<(R > 1)>(r + o);
        }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t row = row0 + q;
      if (row >= rows) break;
      float v[VPL][8];
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int c = (lane + 32 * k) * 8;
        if (lane + 32 * k < nv) {
          rx[q][k].get(v[k]);
          if (r) {
            float t[8];
            rr[q][k].get(t);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[k][e] += t[e];
            Vec8<T>::round(v[k]);   // the stored (rounded) sum is the LN input, as the backward sees it
            Vec8<T>::store(s_out + row * n + c, v[k]);
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) sum += v[k][e];
        }
      }
      const float mean = warp_sum(sum) / float(n);
      float sq = 0.f;
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (lane + 32 * k < nv)
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float d = v[k][e] - mean;
            sq += d * d;
          }
      const float rstd = rsqrtf(warp_sum(sq) / float(n) + eps);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int c = (lane + 32 * k) * 8;
        if (lane + 32 * k < nv) {
          float gg[8], bb[8], o[8];
          Vec8<P>::load(g + c, gg);
          Vec8<P>::load(b + c, bb);
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = (v[k][e] - mean) * rstd * gg[e] + bb[e];
          Vec8<T>::store(y + row * n + c, o);
        }
      }
      if (lane == 0) {
        mean_out[row] = mean;
        rstd_out[row] = rstd;
      }
    }
  }
}

// Backward, pass 1.  Warp w of the grid owns the contiguous rows [w rpw, (w + 1) rpw): per row ds,
// and the warp's partial sums of dy xhat / dy in registers (lane l owns the columns of vectors
// l, l + 32, ...: no atomics, no shared-memory traffic per row); the next row's dy / s are loaded
// while the current one is processed (VPL <= 4).  At the end the block's LN_BWD_WARPS warps are
// combined in warp order and written to part[block][2][n].
constexpr int LN_BWD_WARPS = 12;   // one block per SM: 12 warps x ~140 registers
template <class T, class P, int VPL, bool CS>
__global__ void __launch_bounds__(LN_BWD_WARPS * 32, 1) ln_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ s,
                                                       const P* __restrict__ g, const float* __restrict__ mean_in,
                                                       const float* __restrict__ rstd_in, T* __restrict__ ds,
                                                       float* __restrict__ part, int64_t rows, int n, int64_t rpw) {
  extern __shared__ float acc_sm[];   // [LN_BWD_WARPS][2][n], used once at the end
  constexpr bool PF = VPL <= 4;       // prefetch the next row (register budget)
  const int lane = threadIdx.x & 31;
  const int nv = n >> 3;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t r0 = warp * rpw, r1 = min(rows, r0 + rpw);
  float ag[VPL][8], ab[VPL][8];
#pragma unroll
  for (int k = 0; k < VPL; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) ag[k][e] = ab[k][e] = 0.f;
  Raw8<T> ns[VPL], nd[VPL];   // the next row's s, dy
  float nmean = 0.f, nrstd = 0.f;
  auto fetch = [&](int64_t row) {
    if (row < r1) {
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (lane + 32 * k < nv) {
          ns[k].template load<CS>(s + row * n + (lane + 32 * k) * 8);
          nd[k].template load<CS>(dy + row * n + (lane + 32 * k) * 8);
        }
      nmean = mean_in[row];
      nrstd = rstd_in[row];
    }
  };
  if (PF) fetch(r0);
  for (int64_t row = r0; row < r1; ++row) {
    if (!PF) fetch(row);
    float xh[VPL][8], d[VPL][8];
#pragma unroll
    for (int k = 0; k < VPL; ++k)
      if (lane + 32 * k < nv) {
        ns[k].get(xh[k]);
        nd[k].get(d[k]);
      }
    const float mean = nmean, rstd = nrstd;
    if (PF) fetch(row + 1);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = (lane + 32 * k) * 8;
      if (lane + 32 * k < nv) {
        float gg[8];
        Vec8<P>::load(g + c, gg);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[k][e] = (xh[k][e] - mean) * rstd;
          ag[k][e] += d[k][e] * xh[k][e];
          ab[k][e] += d[k][e];
          d[k][e] *= gg[e];   // dxhat
          s1 += d[k][e];
          s2 += d[k][e] * xh[k][e];
        }
      }
    }
    const float a = warp_sum(s1) / float(n), bq = warp_sum(s2) / float(n);
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = (lane + 32 * k) * 8;
      if (lane + 32 * k < nv) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = rstd * (d[k][e] - a - xh[k][e] * bq);
        Vec8<T>::store(ds + row * n + c, o);
      }
    }
  }
  // the block's warp partials combined in warp order, one partial row pair per block
  float* pg = acc_sm + (threadIdx.x >> 5) * 2 * n;
#pragma unroll
  for (int k = 0; k < VPL; ++k)
    if (lane + 32 * k < nv)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        pg[e * nv + lane + 32 * k] = ag[k][e];   // [e][vector]: conflict-free
        pg[n + e * nv + lane + 32 * k] = ab[k][e];
      }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) {   // column c = vector c / 8, element c % 8
    const int e = (c & 7) * nv + (c >> 3);
    float a = acc_sm[e], b = acc_sm[n + e];
    for (int w = 1; w < LN_BWD_WARPS; ++w) {
      a += acc_sm[w * 2 * n + e];
      b += acc_sm[w * 2 * n + n + e];
    }
    part[(int64_t(blockIdx.x) * 2) * n + c] = a;
    part[(int64_t(blockIdx.x) * 2 + 1) * n + c] = b;
  }
}

// backward, pass 2: dg[c] = sum_w part[w][0][c], db[c] = sum_w part[w][1][c] in a fixed order:
// block (x, y) handles 32 columns of dg (y = 0) or db (y = 1); thread (ty, tx) sums partial rows
// ty, ty + 32, ... then the 32 partials are added in ty order
__global__ void __launch_bounds__(1024) ln_param_reduce_kernel(const float* __restrict__ part, int64_t nw, int n,
                                                              float* __restrict__ dg, float* __restrict__ db) {
  __shared__ float sh[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  const int which = blockIdx.y;
  float a = 0.f;
  if (c < n)
    for (int64_t w = ty; w < nw; w += 32) a += part[(w * 2 + which) * n + c];
  sh[ty][tx] = a;
  __syncthreads();
  if (ty == 0 && c < n) {
    float t = sh[0][tx];
    for (int k = 1; k < 32; ++k) t += sh[k][tx];
    (which ? db : dg)[c] = t;
  }
}

template <class T, class P>
cudaError_t ln_fwd_launch(const void* x, const void* r, const void* g, const void* b, void* y, void* s_out,
                          float* mean, float* rstd, int64_t rows, int n, float eps, cudaStream_t st) {
  const int vpl = (n / 8 + 31) / 32;
  // two rows in flight per warp for bf16 rows when there are enough rows to fill the grid twice
  // over (65 536 x 768: 90 -> 72 us); one below that (8192 x 768: 10.5 vs 12.4 us)
  const bool two = sizeof(T) == 2 && vpl <= 4 && rows >= 32768;
  const int rr = two ? 2 : 1;
  const unsigned blocks = unsigned(std::min<int64_t>((rows + 8 * rr - 1) / (8 * rr), 148 * 8));
#define ROAST_LN_FWD(V)                                                                                         \
  if (two && V <= 4)                                                                                            \
    ln_fwd_kernel<T, P, V, (V <= 4 ? 2 : 1)><<<blocks, 256, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(r),        \
                                                      static_cast<const P*>(g), static_cast<const P*>(b),        \
                                                      static_cast<T*>(y), static_cast<T*>(s_out), mean, rstd,    \
                                                      rows, n, eps);                                             \
  else                                                                                                          \
    ln_fwd_kernel<T, P, V, 1><<<blocks, 256, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(r),        \
                                                      static_cast<const P*>(g), static_cast<const P*>(b),        \
                                                      static_cast<T*>(y), static_cast<T*>(s_out), mean, rstd,    \
                                                      rows, n, eps)
  switch (vpl) {
    case 1: ROAST_LN_FWD(1); break;
    case 2: ROAST_LN_FWD(2); break;
    case 3: ROAST_LN_FWD(3); break;
    case 4: ROAST_LN_FWD(4); break;
    case 5: ROAST_LN_FWD(5); break;
    case 6: ROAST_LN_FWD(6); break;
    case 7: ROAST_LN_FWD(7); break;
    default: ROAST_LN_FWD(8); break;
  }
#undef ROAST_LN_FWD
  return cudaGetLastError();
}

// pass-1 geometry for `rows`: a fixed function of (rows, device SMs), so the reduce order, and
// with it every parameter gradient bit, depends on nothing else
struct LnBwdGrid {
  int64_t rpw, blocks;
};
LnBwdGrid ln_bwd_grid(int64_t rows) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t max_warps = int64_t(sms) * LN_BWD_WARPS;   // one block per SM
  const int64_t rpw = std::max<int64_t>(1, (rows + max_warps - 1) / max_warps);
  const int64_t warps = std::max<int64_t>(1, (rows + rpw - 1) / rpw);
  return {rpw, (warps + LN_BWD_WARPS - 1) / LN_BWD_WARPS};
}

template <class T, class P>
cudaError_t ln_bwd_launch(const void* dy, const void* s, const void* g, const float* mean, const float* rstd, void* ds,
                          float* part, const LnBwdGrid& gr, int64_t rows, int n, cudaStream_t st) {
  const int vpl = (n / 8 + 31) / 32;
  const size_t smem = 2 * LN_BWD_WARPS * size_t(n) * sizeof(float);   // per warp (dg, db) partials
  const bool cs = rows >= 32768;   // inputs not L2-resident: streaming loads
  // the smem opt-in once per instantiation and device (at the largest n), not on every call
#define ROAST_LN_BWD_CS(V, CSV)                                                                                \
  {                                                                                                             \
    static std::atomic<unsigned long long> opted{0};                                                            \
    if (first_on_device(opted))                                                                                 \
      cudaFuncSetAttribute(ln_bwd_kernel<T, P, V, CSV>, cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                           int(2 * LN_BWD_WARPS * 2048 * sizeof(float)));                                       \
  }                                                                                                             \
  ln_bwd_kernel<T, P, V, CSV><<<unsigned(gr.blocks), LN_BWD_WARPS * 32, smem, st>>>(                           \
      static_cast<const T*>(dy), static_cast<const T*>(s), static_cast<const P*>(g), mean, rstd,               \
      static_cast<T*>(ds), part, rows, n, gr.rpw)
#define ROAST_LN_BWD(V)       \
  if (cs) {                   \
    ROAST_LN_BWD_CS(V, true);  \
  } else {                    \
    ROAST_LN_BWD_CS(V, false); \
  }
  switch (vpl) {
    case 1: ROAST_LN_BWD(1); break;
    case 2: ROAST_LN_BWD(2); break;
    case 3: ROAST_LN_BWD(3); break;
    case 4: ROAST_LN_BWD(4); break;
    case 5: ROAST_LN_BWD(5); break;
    case 6: ROAST_LN_BWD(6); break;
    case 7: ROAST_LN_BWD(7); break;
    default: ROAST_LN_BWD(8); break;
  }
#undef ROAST_LN_BWD
#undef ROAST_LN_BWD_CS
  return cudaGetLastError();
}

}  // namespace
}  // namespace roast

using namespace roast;

extern "C" {

roast_status_t roast_layernorm_fwd(const void* x, const void* r, const void* gamma, const void* beta, void* y,
                                   void* s_out, float* mean, float* rstd, int64_t rows, int32_t n, float eps,
                                   roast_dtype_t dt, roast_dtype_t pdt, roast_stream_t stream) {
  if (rows < 0 || n <= 0 || n % 8 || n > 2048) return fail(ROAST_ERR_SHAPE, "layernorm: n % 8 == 0, 8 <= n <= 2048");
  if (!x || !gamma || !beta || !y || !mean || !rstd || (r && !s_out))
    return fail(ROAST_ERR_CONFIG, "layernorm: null pointer (s_out is required with a residual)");
  if (rows == 0) return ROAST_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (dt == ROAST_BF16 && pdt == ROAST_BF16)
    e = ln_fwd_launch<__nv_bfloat16, __nv_bfloat16>(x, r, gamma, beta, y, s_out, mean, rstd, rows, n, eps, s);
  else if (dt == ROAST_BF16)
    e = ln_fwd_launch<__nv_bfloat16, float>(x, r, gamma, beta, y, s_out, mean, rstd, rows, n, eps, s);
  else if (pdt == ROAST_BF16)
    e = ln_fwd_launch<float, __nv_bfloat16>(x, r, gamma, beta, y, s_out, mean, rstd, rows, n, eps, s);
  else
    e = ln_fwd_launch<float, float>(x, r, gamma, beta, y, s_out, mean, rstd, rows, n, eps, s);
  ROAST_CUDA_CHECK(e);
  return ROAST_OK;
}

roast_status_t roast_layernorm_bwd(const void* dy, const void* s_in, const void* gamma, const float* mean,
                                   const float* rstd, void* ds, float* dgamma, float* dbeta, int64_t rows, int32_t n,
                                   roast_dtype_t dt, roast_dtype_t pdt, roast_stream_t stream) {
  if (rows < 0 || n <= 0 || n % 8 || n > 2048) return fail(ROAST_ERR_SHAPE, "layernorm: n % 8 == 0, 8 <= n <= 2048");
  if (!dy || !s_in || !gamma || !mean || !rstd || !ds || !dgamma || !dbeta)
    return fail(ROAST_ERR_CONFIG, "layernorm: null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // pass 1's grid is a fixed function of the row count (ln_bwd_grid): the reduce order is
  // data-independent; each block leaves 2 n partials
  if (rows == 0) {
    ROAST_CUDA_CHECK(cudaMemsetAsync(dgamma, 0, size_t(n) * sizeof(float), s));
    ROAST_CUDA_CHECK(cudaMemsetAsync(dbeta, 0, size_t(n) * sizeof(float), s));
    return ROAST_OK;
  }
  const LnBwdGrid gr = ln_bwd_grid(rows);
  Scratch ws;
  if (roast_status_t st = scratch_alloc(ws, size_t(gr.blocks) * 2 * size_t(n) * sizeof(float), s)) return st;
  cudaError_t e;
  if (dt == ROAST_BF16 && pdt == ROAST_BF16)
    e = ln_bwd_launch<__nv_bfloat16, __nv_bfloat16>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), gr, rows, n, s);
  else if (dt == ROAST_BF16)
    e = ln_bwd_launch<__nv_bfloat16, float>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), gr, rows, n, s);
  else if (pdt == ROAST_BF16)
    e = ln_bwd_launch<float, __nv_bfloat16>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), gr, rows, n, s);
  else
    e = ln_bwd_launch<float, float>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), gr, rows, n, s);
  ROAST_CUDA_CHECK(e);
  ln_param_reduce_kernel<<<dim3(unsigned((n + 31) / 32), 2), 1024, 0, s>>>(ws.as<float>(), gr.blocks, n, dgamma, dbeta);
  ROAST_CUDA_CHECK(cudaGetLastError());
  return ROAST_OK;
}

}  // extern "C"
