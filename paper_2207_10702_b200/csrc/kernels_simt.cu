// kernels_simt.cu — SIMT (FFMA) ROAST-MM for any hash-tile geometry (K1), the
// deterministic dM segmented reduce (K5), shadow refresh / SGD (K8), and the
// recovered-weight debug hook.
//
// ROAST-MM, Algorithm 1: every Z1 x Z2 tile of the virtual
// weight W is read from M at offset h2(x, y), element (o1, o2) at pi(o1, o2)
// (P:284), multiplied by the tile sign g; the output tile is scaled by
// lambda once after the k-accumulation.  Backward: dX
// through the same tiles transposed; dW tiles scattered into dM with lambda * g.
#include <cuda_bf16.h>

#include "roast_internal.h"

namespace roast {
namespace {

__device__ __forceinline__ int pi_index(int o1, int o2, int z2, int layout) {
  if (layout == ROAST_SW128) return z2 * o1 + 8 * ((o2 >> 3) ^ (o1 & 7)) + (o2 & 7);
  return z2 * o1 + o2;
}

struct MapArgs {
  const int64_t* off;
  const int8_t* sgn;
  int z1, z2, ny, layout;
  int64_t neg_base;  // bf16 shadow: index of the negated copy
};

template <typename T>
__device__ __forceinline__ float load_val(const T* p, int64_t i);
template <>
__device__ __forceinline__ float load_val<float>(const float* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ float load_val<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
template <typename T>
__device__ __forceinline__ void store_val(T* p, int64_t i, float v);
template <>
__device__ __forceinline__ void store_val<float>(float* p, int64_t i, float v) { p[i] = v; }
template <>
__device__ __forceinline__ void store_val<__nv_bfloat16>(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

// Recovered (unscaled, signed) weight W~[h][o] = g * Mop[off + pi].
template <typename MT>
__device__ __forceinline__ float wtile(const MT* Mop, const MapArgs& a, int h, int o) {
  int x = h / a.z1, y = o / a.z2;
  int t = x * a.ny + y;
  int64_t slot = a.off[t] + pi_index(h - x * a.z1, o - y * a.z2, a.z2, a.layout);
  float v = load_val(Mop, slot);
  return a.sgn[t] < 0 ? -v : v;
}

constexpr int BM = 64, BN = 64, BK = 16;

// C[T x N] = lam * A[T x K] * B[K x N]; B[k][n] = W~[k][n] (fwd) or W~[n][k] (dX).
template <typename XT, typename MT, bool kTransW>
__global__ void __launch_bounds__(256) simt_mm_kernel(const XT* __restrict__ A, XT* __restrict__ C,
                                                      const MT* __restrict__ Mop, MapArgs map, int64_t T,
                                                      int K, int N, float lam, const float* __restrict__ bias) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  const int64_t m0 = int64_t(blockIdx.y) * BM;
  const int n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = tid; e < BM * BK; e += 256) {
      int r = e / BK, kk = e % BK;
      int64_t m = m0 + r;
      int k = k0 + kk;
      As[kk][r] = (m < T && k < K) ? load_val(A, m * K + k) : 0.f;
    }
    for (int e = tid; e < BK * BN; e += 256) {
      int kk = e / BN, nn = e % BN;
      int k = k0 + kk, n = n0 + nn;
      float v = 0.f;
      if (k < K && n < N) v = kTransW ? wtile(Mop, map, n, k) : wtile(Mop, map, k, n);
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tr * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tc * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + tr * 4 + i;
    if (m >= T) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tc * 4 + j;
      if (n < N) store_val(C, m * N + n, bias ? fmaf(lam, acc[i][j], bias[n]) : lam * acc[i][j]);
    }
  }
}

// G[H x O] = X^T dY (K = tokens); epilogue scatters lam * g * G into its hash tile:
// ws[(x*ny + y) * Z1Z2 + pi] (deterministic, reduced by K5) or atomically into dM.
template <typename XT>
__global__ void __launch_bounds__(256) simt_dw_kernel(const XT* __restrict__ X, const XT* __restrict__ dY,
                                                      MapArgs map, int64_t T, int H, int O, float lam,
                                                      float* __restrict__ ws, float* __restrict__ dM) {
  __shared__ float Xs[BK][BM + 4];
  __shared__ float Ds[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  const int h0 = blockIdx.y * BM;
  const int o0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int64_t t0 = 0; t0 < T; t0 += BK) {
    for (int e = tid; e < BK * BM; e += 256) {
      int kk = e / BM, r = e % BM;
      int64_t t = t0 + kk;
      Xs[kk][r] = (t < T && h0 + r < H) ? load_val(X, t * H + h0 + r) : 0.f;
      Ds[kk][r] = (t < T && o0 + r < O) ? load_val(dY, t * O + o0 + r) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Xs[kk][tr * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ds[kk][tc * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int tile_elems = map.z1 * map.z2;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int h = h0 + tr * 4 + i;
    if (h >= H) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int o = o0 + tc * 4 + j;
      if (o >= O) continue;
      int x = h / map.z1, y = o / map.z2;
      int t = x * map.ny + y;
      int p = pi_index(h - x * map.z1, o - y * map.z2, map.z2, map.layout);
      float v = lam * (map.sgn[t] < 0 ? -acc[i][j] : acc[i][j]);
      if (ws)
        ws[int64_t(t) * tile_elems + p] = v;
      else
        atomicAdd(dM + map.off[t] + p, v);
    }
  }
}

// K5: dM[s] += sum over covering tiles (ascending (offset, tile id)), then over
// split-K partials (ascending), of ws[split][tile][s - off].  One thread per
// 4 consecutive slots; A % 4 == 0 and T % A == 0 so all 4 share one covering set.
__global__ void det_reduce_kernel(float* __restrict__ dM, const float* __restrict__ ws,
                                  const int32_t* __restrict__ sorted, const int64_t* __restrict__ sorted_off,
                                  int ntiles, int64_t tile_elems, int nsplit, int64_t mem_size) {
  int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t s = q * 4;
  if (s >= mem_size) return;
  // lo = first i with sorted_off[i] > s - T ; hi = first i with sorted_off[i] > s
  int lo = 0, hi = ntiles;
  {
    int64_t key = s - tile_elems;
    int a = 0, b = ntiles;
    while (a < b) { int mid = (a + b) >> 1; if (sorted_off[mid] > key) b = mid; else a = mid + 1; }
    lo = a;
    a = lo; b = ntiles;
    while (a < b) { int mid = (a + b) >> 1; if (sorted_off[mid] > s) b = mid; else a = mid + 1; }
    hi = a;
  }
  if (lo >= hi) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t split_stride = int64_t(ntiles) * tile_elems;
  for (int i = lo; i < hi; ++i) {
    int64_t base = int64_t(sorted[i]) * tile_elems + (s - sorted_off[i]);
    for (int sp = 0; sp < nsplit; ++sp) {
      float4 v = *reinterpret_cast<const float4*>(ws + sp * split_stride + base);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  float4* d = reinterpret_cast<float4*>(dM + s);
  float4 o = *d;
  o.x += acc.x; o.y += acc.y; o.z += acc.z; o.w += acc.w;
  *d = o;
}

__global__ void sync_shadow_kernel(const float* __restrict__ M, __nv_bfloat16* __restrict__ sh, int64_t n,
                                   int64_t neg_base) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    __nv_bfloat16 b = __float2bfloat16_rn(M[i]);
    sh[i] = b;
    sh[neg_base + i] = __hneg(b);
  }
}

__global__ void sgd_kernel(float* __restrict__ M, const float* __restrict__ dM, __nv_bfloat16* __restrict__ sh,
                           int64_t n, int64_t neg_base, float lr) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float v = M[i] - lr * dM[i];
    M[i] = v;
    __nv_bfloat16 b = __float2bfloat16_rn(v);
    sh[i] = b;
    sh[neg_base + i] = __hneg(b);
  }
}

__global__ void materialize_kernel(const float* __restrict__ M, const __nv_bfloat16* __restrict__ sh, MapArgs map,
                                   int H, int O, float lam, int bf16_out, void* W) {
  int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= int64_t(H) * O) return;
  int h = int(e / O), o = int(e % O);
  int x = h / map.z1, y = o / map.z2;
  int t = x * map.ny + y;
  int64_t slot = map.off[t] + pi_index(h - x * map.z1, o - y * map.z2, map.z2, map.layout);
  if (bf16_out) {
    // the tensor-core operand: read from the + or - half of the shadow
    reinterpret_cast<__nv_bfloat16*>(W)[e] = sh[map.sgn[t] < 0 ? map.neg_base + slot : slot];
  } else {
    float v = __fmul_rn(lam, M[slot]);
    reinterpret_cast<float*>(W)[e] = map.sgn[t] < 0 ? -v : v;
  }
}

MapArgs map_args(const Ctx* c, const Module& m) {
  MapArgs a;
  a.off = m.d_off;
  a.sgn = m.d_sgn;
  a.z1 = c->tile.z1;
  a.z2 = c->tile.z2;
  a.ny = m.ny;
  a.layout = c->cfg.tile_layout;
  a.neg_base = c->neg_base;
  return a;
}

int grid_1d(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return int(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_simt_fwd(const Ctx* c, const Module& m, const void* X, void* Y, int64_t T, roast_dtype_t dt,
                            bool transpose_w, cudaStream_t s, const float* bias) {
  if (T == 0) return cudaSuccess;
  const int K = int(transpose_w ? m.O : m.H);
  const int N = int(transpose_w ? m.H : m.O);
  dim3 grid((N + BN - 1) / BN, unsigned((T + BM - 1) / BM));
  MapArgs a = map_args(c, m);
  if (dt == ROAST_FP32) {
    if (transpose_w)
      simt_mm_kernel<float, float, true><<<grid, 256, 0, s>>>((const float*)X, (float*)Y, c->M, a, T, K, N, m.lam, bias);
    else
      simt_mm_kernel<float, float, false><<<grid, 256, 0, s>>>((const float*)X, (float*)Y, c->M, a, T, K, N, m.lam, bias);
  } else {
    auto* sh = reinterpret_cast<const __nv_bfloat16*>(c->shadow);
    if (transpose_w)
      simt_mm_kernel<__nv_bfloat16, __nv_bfloat16, true>
          <<<grid, 256, 0, s>>>((const __nv_bfloat16*)X, (__nv_bfloat16*)Y, sh, a, T, K, N, m.lam, bias);
    else
      simt_mm_kernel<__nv_bfloat16, __nv_bfloat16, false>
          <<<grid, 256, 0, s>>>((const __nv_bfloat16*)X, (__nv_bfloat16*)Y, sh, a, T, K, N, m.lam, bias);
  }
  return cudaGetLastError();
}

cudaError_t launch_simt_dw(const Ctx* c, const Module& m, const void* X, const void* dY, int64_t T,
                           roast_dtype_t dt, float* ws, cudaStream_t s) {
  dim3 grid(unsigned((m.O + BN - 1) / BN), unsigned((m.H + BM - 1) / BM));
  MapArgs a = map_args(c, m);
  if (dt == ROAST_FP32)
    simt_dw_kernel<float><<<grid, 256, 0, s>>>((const float*)X, (const float*)dY, a, T, int(m.H), int(m.O), m.lam,
                                               ws, c->dM);
  else
    simt_dw_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)X, (const __nv_bfloat16*)dY, a, T,
                                                       int(m.H), int(m.O), m.lam, ws, c->dM);
  return cudaGetLastError();
}

cudaError_t launch_det_reduce(const Ctx* c, const Module& m, const float* ws, int nsplit, cudaStream_t s) {
  int64_t nthreads = c->mem_size / 4;
  int threads = 256;
  int64_t blocks = (nthreads + threads - 1) / threads;
  det_reduce_kernel<<<unsigned(blocks), threads, 0, s>>>(c->dM, ws, m.d_sorted, m.d_sorted_off, m.nx * m.ny,
                                                         int64_t(c->tile.z1) * c->tile.z2, nsplit, c->mem_size);
  return cudaGetLastError();
}

cudaError_t launch_sync_shadow(Ctx* c, cudaStream_t s) {
  sync_shadow_kernel<<<grid_1d(c->mem_size, 256), 256, 0, s>>>(
      c->M, reinterpret_cast<__nv_bfloat16*>(c->shadow), c->mem_size, c->neg_base);
  return cudaGetLastError();
}

cudaError_t launch_sgd(Ctx* c, float lr, cudaStream_t s) {
  sgd_kernel<<<grid_1d(c->mem_size, 256), 256, 0, s>>>(c->M, c->dM, reinterpret_cast<__nv_bfloat16*>(c->shadow),
                                                       c->mem_size, c->neg_base, lr);
  return cudaGetLastError();
}

cudaError_t launch_materialize(const Ctx* c, const Module& m, roast_dtype_t dt, void* W, cudaStream_t s) {
  int64_t n = m.H * m.O;
  if (n == 0) return cudaSuccess;
  materialize_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(
      c->M, reinterpret_cast<const __nv_bfloat16*>(c->shadow), map_args(c, m), int(m.H), int(m.O), m.lam,
      dt == ROAST_BF16, W);
  return cudaGetLastError();
}

}  // namespace roast

namespace roast {
namespace {

// One pass over |M|: update M from dM (and the optimizer state), refresh both halves of the
// bf16 shadow, optionally zero dM.  kind: 0 SGD, 1 Adagrad, 2 Adam (PyTorch formulas).
template <int KIND>
__global__ void opt_kernel(float* __restrict__ M, float* __restrict__ dM, __nv_bfloat16* __restrict__ sh,
                           float* __restrict__ s1, float* __restrict__ s2, int64_t n, int64_t neg_base, float lr,
                           float b1, float b2, float eps, float wd, float bc1, float bc2, int zero) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float w = M[i];
    const float g = dM[i] + wd * w;
    if (KIND == 0) {
      w -= lr * g;
    } else if (KIND == 1) {
      const float G = s1[i] + g * g;
      s1[i] = G;
      w -= lr * g / (sqrtf(G) + eps);
    } else {
      const float m = b1 * s1[i] + (1.f - b1) * g;
      const float v = b2 * s2[i] + (1.f - b2) * g * g;
      s1[i] = m;
      s2[i] = v;
      w -= lr * (m / bc1) / (sqrtf(v / bc2) + eps);
    }
    M[i] = w;
    const __nv_bfloat16 b = __float2bfloat16_rn(w);
    sh[i] = b;
    sh[neg_base + i] = __hneg(b);
    if (zero) dM[i] = 0.f;
  }
}

}  // namespace

cudaError_t launch_optimizer(Ctx* c, int kind, float lr, float b1, float b2, float eps, float wd, int64_t step,
                             int zero, cudaStream_t s) {
  const float bc1 = kind == 2 ? float(1.0 - pow(double(b1), double(step))) : 1.f;
  const float bc2 = kind == 2 ? float(1.0 - pow(double(b2), double(step))) : 1.f;
  auto* sh = reinterpret_cast<__nv_bfloat16*>(c->shadow);
  const int grid = grid_1d(c->mem_size, 256);
  if (kind == 0)
    opt_kernel<0><<<grid, 256, 0, s>>>(c->M, c->dM, sh, nullptr, nullptr, c->mem_size, c->neg_base, lr, b1, b2, eps,
                                       wd, bc1, bc2, zero);
  else if (kind == 1)
    opt_kernel<1><<<grid, 256, 0, s>>>(c->M, c->dM, sh, c->opt_s1, nullptr, c->mem_size, c->neg_base, lr, b1, b2,
                                       eps, wd, bc1, bc2, zero);
  else
    opt_kernel<2><<<grid, 256, 0, s>>>(c->M, c->dM, sh, c->opt_s1, c->opt_s2, c->mem_size, c->neg_base, lr, b1, b2,
                                       eps, wd, bc1, bc2, zero);
  return cudaGetLastError();
}

}  // namespace roast
