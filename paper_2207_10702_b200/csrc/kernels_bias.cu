// kernels_bias.cu — the column sum behind a bias recovered with L (NEXT #3).
//
// A bias vector b of n elements is row 0 of a 1 x n ROAST embedding ("ROAST uses
// L to implement ... bias vectors").  Its forward is the L lookup, added to Y inside the
// forward GEMM's epilogue (gemm_sm100.cu / kernels_simt.cu).  Its backward is
//     db[j] = sum_t dY[t, j]          (this file: fp32, fixed summation order)
//     dM[h1(c) + o] += lambda g(c) db[jZ + o]      (the L backward, kernels_embed*.cu)
//
// Mapping to the machine: HBM-bound streaming read of dY.  A CTA owns 64 columns x one
// slab of rows; each warp reads whole 128-B (bf16) / 256-B (fp32) row segments, lane l
// accumulating columns 2l, 2l+1 in fp32 over rows warp, warp + 8, ...; the 8 warps are
// combined in warp order, the slabs by a second tiny kernel in slab order, so the result
// is bitwise reproducible.  Grid = column blocks x slabs ~ 2 waves of 148 SMs.
#include <cuda_bf16.h>

#include "roast_internal.h"

namespace roast {
namespace {

template <typename XT>
__global__ void __launch_bounds__(256) colsum_kernel(const XT* __restrict__ dY, int64_t T, int n, int64_t ld,
                                                     int64_t rows_per_slab, float* __restrict__ partial) {
  __shared__ float2 red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = blockIdx.x * 64 + 2 * lane;
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_slab;
  const int64_t r1 = min(T, r0 + rows_per_slab);
  float2 acc = make_float2(0.f, 0.f);
  if (col < n) {
    int64_t r = r0 + warp;
    for (; r + 24 < r1; r += 32) {   // 4 independent rows in flight per warp
      float2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if constexpr (sizeof(XT) == 2) {
          const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(dY + (r + 8 * u) * ld + col);
          v[u] = __bfloat1622float2(b);
        } else {
          v[u] = *reinterpret_cast<const float2*>(dY + (r + 8 * u) * ld + col);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
      }
    }
    for (; r < r1; r += 8) {
      float2 v;
      if constexpr (sizeof(XT) == 2)
        v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dY + r * ld + col));
      else
        v = *reinterpret_cast<const float2*>(dY + r * ld + col);
      acc.x += v.x;
      acc.y += v.y;
    }
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && col < n) {
    float2 s = red[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      s.x += red[w][lane].x;
      s.y += red[w][lane].y;
    }
    *reinterpret_cast<float2*>(partial + int64_t(blockIdx.y) * n + col) = s;
  }
}

__global__ void slab_sum_kernel(const float* __restrict__ partial, int slabs, int n, float* __restrict__ db,
                                int accumulate) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float s = 0.f;
  for (int k = 0; k < slabs; ++k) s += partial[int64_t(k) * n + j];
  db[j] = accumulate ? db[j] + s : s;
}

}  // namespace

int colsum_slabs(int64_t T, int n) {
  const int64_t cb = (n + 63) / 64;
  int64_t slabs = (296 + cb - 1) / cb;                 // ~2 CTAs per SM
  slabs = std::min<int64_t>(slabs, (T + 255) / 256);   // >= 256 rows per slab
  return int(std::max<int64_t>(slabs, 1));
}

cudaError_t launch_colsum(const void* dY, int64_t T, int n, int64_t ld, roast_dtype_t dt, float* partial, float* db,
                          cudaStream_t s, int accumulate) {
  const int slabs = colsum_slabs(T, n);
  const int64_t rows = (T + slabs - 1) / slabs;
  dim3 grid(unsigned((n + 63) / 64), unsigned(slabs));
  if (dt == ROAST_BF16)
    colsum_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dY), T, n, ld, rows, partial);
  else
    colsum_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(dY), T, n, ld, rows, partial);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  slab_sum_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(partial, slabs, n, db, accumulate);
  return cudaGetLastError();
}

}  // namespace roast
