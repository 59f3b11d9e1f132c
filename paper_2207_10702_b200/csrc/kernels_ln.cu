// kernels_ln.cu — LayerNorm of the ROASTed BERT workload: the
// N-operations stay plain, but at C3's 65 536 tokens torch's LayerNorm spends 0.85 ms
// per call (its parameter-gradient kernel alone 0.56 ms), more than the layer's ROAST GEMMs.
// Here one pass each way, memory-bound:
//   forward  : s = x (+ r, the residual, fused), mean / rstd per row, y = (s - mean) rstd g + b
//   backward : xhat = (s - mean) rstd, dxhat = dy g,
//              ds = rstd (dxhat - mean(dxhat) - xhat mean(dxhat xhat)),
//              dg = sum_rows dy xhat, db = sum_rows dy  (per-warp partials, then a fixed-order
//              reduce: bitwise reproducible)
// One warp per row; lane l holds the 8-element vectors l, l + 32, ... of the row in registers.
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

template <class T, class P, int VPL>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const T* __restrict__ x, const T* __restrict__ r,
                                                    const P* __restrict__ g, const P* __restrict__ b,
                                                    T* __restrict__ y, T* __restrict__ s_out,
                                                    float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                    int64_t rows, int n, float eps) {
  const int lane = threadIdx.x & 31;
  const int nv = n >> 3;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < rows; row += nwarps) {
    float v[VPL][8];
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = (lane + 32 * k) * 8;
      if (lane + 32 * k < nv) {
        Vec8<T>::load(x + row * n + c, v[k]);
        if (r) {
          float t[8];
          Vec8<T>::load(r + row * n + c, t);
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

// backward, pass 1: ds per row, and per-warp partial sums of dy xhat / dy over the warp's rows
// (rows w, w + nwarps, ... in that order), kept in the warp's slice of shared memory (each lane
// owns its columns: no atomics); at the end the block's 8 warps are combined in warp order and
// written to part[block][2][n]
template <class T, class P, int VPL>
__global__ void __launch_bounds__(256) ln_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ s,
                                                    const P* __restrict__ g, const float* __restrict__ mean_in,
                                                    const float* __restrict__ rstd_in, T* __restrict__ ds,
                                                    float* __restrict__ part, int64_t rows, int n) {
  extern __shared__ float acc_sm[];   // [8 warps][2][n]
  const int lane = threadIdx.x & 31;
  const int nv = n >> 3;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  float* pg = acc_sm + (threadIdx.x >> 5) * 2 * n;
  float* pb = pg + n;
  for (int c = lane; c < n; c += 32) {
    pg[c] = 0.f;
    pb[c] = 0.f;
  }
  __syncwarp();
  for (int64_t row = warp; row < rows; row += nwarps) {
    const float mean = mean_in[row], rstd = rstd_in[row];
    float xh[VPL][8], d[VPL][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = (lane + 32 * k) * 8;
      if (lane + 32 * k < nv) {
        Vec8<T>::load(s + row * n + c, xh[k]);
        Vec8<T>::load(dy + row * n + c, d[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int c = (lane + 32 * k) * 8;
      if (lane + 32 * k < nv) {
        float gg[8];
        Vec8<P>::load(g + c, gg);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[k][e] = (xh[k][e] - mean) * rstd;
          pg[e * nv + lane + 32 * k] += d[k][e] * xh[k][e];   // [e][vector]: conflict-free
          pb[e * nv + lane + 32 * k] += d[k][e];
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
  // the block's 8 warp partials combined in warp order, one partial row pair per block
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) {   // column c = vector c / 8, element c % 8
    const int e = (c & 7) * nv + (c >> 3);
    float a = acc_sm[e], b = acc_sm[n + e];
    for (int w = 1; w < 8; ++w) {
      a += acc_sm[w * 2 * n + e];
      b += acc_sm[w * 2 * n + n + e];
    }
    part[(int64_t(blockIdx.x) * 2) * n + c] = a;
    part[(int64_t(blockIdx.x) * 2 + 1) * n + c] = b;
  }
}

// backward, pass 2: dg[c] = sum_w part[w][0][c], db[c] = sum_w part[w][1][c] in a fixed order:
// thread (ty, tx) of a 32-column block (32 x 32 threads) sums warps ty, ty + 32, ... then the 32
// partials are added in ty order
__global__ void __launch_bounds__(1024) ln_param_reduce_kernel(const float* __restrict__ part, int64_t nw, int n,
                                                              float* __restrict__ dg, float* __restrict__ db) {
  __shared__ float sh[2][32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float a = 0.f, b = 0.f;
  if (c < n)
    for (int64_t w = ty; w < nw; w += 32) {
      a += part[(w * 2) * n + c];
      b += part[(w * 2 + 1) * n + c];
    }
  sh[0][ty][tx] = a;
  sh[1][ty][tx] = b;
  __syncthreads();
  if (ty == 0 && c < n) {
    float ta = sh[0][0][tx], tb = sh[1][0][tx];
    for (int k = 1; k < 32; ++k) {
      ta += sh[0][k][tx];
      tb += sh[1][k][tx];
    }
    dg[c] = ta;
    db[c] = tb;
  }
}

template <class T, class P>
cudaError_t ln_fwd_launch(const void* x, const void* r, const void* g, const void* b, void* y, void* s_out,
                          float* mean, float* rstd, int64_t rows, int n, float eps, cudaStream_t st) {
  const int vpl = (n / 8 + 31) / 32;
  const unsigned blocks = unsigned(std::min<int64_t>((rows + 7) / 8, 148 * 16));
#define ROAST_LN_FWD(V)                                                                                         \
  ln_fwd_kernel<T, P, V><<<blocks, 256, 0, st>>>(static_cast<const T*>(x), static_cast<const T*>(r),             \
                                                 static_cast<const P*>(g), static_cast<const P*>(b),             \
                                                 static_cast<T*>(y), static_cast<T*>(s_out), mean, rstd, rows, n, eps)
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

template <class T, class P>
cudaError_t ln_bwd_launch(const void* dy, const void* s, const void* g, const float* mean, const float* rstd, void* ds,
                          float* part, int64_t nw, int64_t rows, int n, cudaStream_t st) {
  const int vpl = (n / 8 + 31) / 32;
  const unsigned blocks = unsigned(nw / 8);
  const size_t smem = 16 * size_t(n) * sizeof(float);   // 8 warps x (dg, db) partials
#define ROAST_LN_BWD(V)                                                                                        \
  cudaFuncSetAttribute(ln_bwd_kernel<T, P, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));          \
  ln_bwd_kernel<T, P, V><<<blocks, 256, smem, st>>>(static_cast<const T*>(dy), static_cast<const T*>(s),           \
                                                 static_cast<const P*>(g), mean, rstd, static_cast<T*>(ds), part, \
                                                 rows, n)
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
  // warps of pass 1 (a fixed grid for a given row count: the reduce order is data-independent);
  // each leaves 2 n partials
  // ~4 rows per warp, at most one resident wave of 148 x 4 blocks; the reduce reads one partial
  // row pair per block
  const int64_t nw = std::max<int64_t>(8, std::min<int64_t>((rows / 4 + 7) / 8 * 8, int64_t(148) * 4 * 8));
  Scratch ws;
  if (roast_status_t st = scratch_alloc(ws, size_t(nw / 8) * 2 * size_t(n) * sizeof(float), s)) return st;
  cudaError_t e;
  if (dt == ROAST_BF16 && pdt == ROAST_BF16)
    e = ln_bwd_launch<__nv_bfloat16, __nv_bfloat16>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), nw, rows, n, s);
  else if (dt == ROAST_BF16)
    e = ln_bwd_launch<__nv_bfloat16, float>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), nw, rows, n, s);
  else if (pdt == ROAST_BF16)
    e = ln_bwd_launch<float, __nv_bfloat16>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), nw, rows, n, s);
  else
    e = ln_bwd_launch<float, float>(dy, s_in, gamma, mean, rstd, ds, ws.as<float>(), nw, rows, n, s);
  ROAST_CUDA_CHECK(e);
  ln_param_reduce_kernel<<<unsigned((n + 31) / 32), 1024, 0, s>>>(ws.as<float>(), nw / 8, n, dgamma, dbeta);
  ROAST_CUDA_CHECK(cudaGetLastError());
  return ROAST_OK;
}

}  // extern "C"
