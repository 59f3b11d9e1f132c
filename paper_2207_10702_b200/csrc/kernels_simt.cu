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

// BK = 64: the hashed B gathers (tile map -> M, two dependent loads) of a whole 64-deep
// K slice are in flight at once; with BK = 16 the small fp32 configs (C1: 4 blocks) were
// bound by 16 serial load-latency rounds.
constexpr int BK = 64;

// C[T x N] = lam * A[T x K] * B[K x N]; B[k][n] = W~[k][n] (fwd) or W~[n][k] (dX).
template <typename XT, typename MT, bool kTransW, int TS>
__global__ void __launch_bounds__(256) simt_mm_kernel(const XT* __restrict__ A, XT* __restrict__ C,
                                                      const MT* __restrict__ Mop, MapArgs map, int64_t T,
                                                      int K, int N, float lam, const float* __restrict__ bias) {
  constexpr int BM = TS, BN = TS, RM = TS / 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  const int64_t m0 = int64_t(blockIdx.y) * BM;
  const int n0 = blockIdx.x * BN;
  float acc[RM][RM] = {};
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
      float a[RM], b[RM];
#pragma unroll
      for (int i = 0; i < RM; ++i) a[i] = As[kk][tr * RM + i];
#pragma unroll
      for (int j = 0; j < RM; ++j) b[j] = Bs[kk][tc * RM + j];
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RM; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    int64_t m = m0 + tr * RM + i;
    if (m >= T) continue;
#pragma unroll
    for (int j = 0; j < RM; ++j) {
      int n = n0 + tc * RM + j;
      if (n < N) store_val(C, m * N + n, bias ? fmaf(lam, acc[i][j], bias[n]) : lam * acc[i][j]);
    }
  }
}

// G[H x O] = X^T dY (K = tokens); epilogue scatters lam * g * G into its hash tile:
// ws[(x*ny + y) * Z1Z2 + pi] (deterministic, reduced by K5) or atomically into dM.
template <typename XT, int TS>
__global__ void __launch_bounds__(256) simt_dw_kernel(const XT* __restrict__ X, const XT* __restrict__ dY,
                                                      MapArgs map, int64_t T, int H, int O, float lam,
                                                      float* __restrict__ ws, float* __restrict__ dM) {
  constexpr int BM = TS, BN = TS, RM = TS / 16;
  __shared__ float Xs[BK][BM + 4];
  __shared__ float Ds[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  const int h0 = blockIdx.y * BM;
  const int o0 = blockIdx.x * BN;
  float acc[RM][RM] = {};
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
      float a[RM], b[RM];
#pragma unroll
      for (int i = 0; i < RM; ++i) a[i] = Xs[kk][tr * RM + i];
#pragma unroll
      for (int j = 0; j < RM; ++j) b[j] = Ds[kk][tc * RM + j];
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RM; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int tile_elems = map.z1 * map.z2;
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    int h = h0 + tr * RM + i;
    if (h >= H) continue;
#pragma unroll
    for (int j = 0; j < RM; ++j) {
      int o = o0 + tc * RM + j;
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
// Visited slots: every 4-slot group of |M| (n_iv == 0), or only the touched set (the exchange's
// interval tables, exchange.cu): slot groups no tile covers are skipped without a search,
// which at |M| >> n (C5: 512 M slots, 16.5 M touched) is most of the pass.
__global__ void det_reduce_kernel(float* __restrict__ dM, const float* __restrict__ ws,
                                  const int32_t* __restrict__ sorted, const int64_t* __restrict__ sorted_off,
                                  int ntiles, int64_t tile_elems, int nsplit, int64_t mem_size,
                                  const int64_t* __restrict__ iv_start, const int64_t* __restrict__ iv_prefix,
                                  int n_iv, int64_t n_touched) {
  // each CTA takes a contiguous range of slot groups; a thread's slots increase, so the
  // touched interval and the covering tile range [lo, hi) are found by binary search once and
  // then only advanced (the summation order per slot is unchanged)
  const int64_t n = n_iv > 0 ? n_touched : mem_size;
  int64_t b, e;
  cta_range(n, 4, &b, &e);
  IvWalk walk{iv_start, iv_prefix, n_iv};
  int lo = -1, hi = 0;
  const int64_t split_stride = int64_t(ntiles) * tile_elems;
  for (int64_t p = b + int64_t(threadIdx.x) * 4; p < e; p += int64_t(blockDim.x) * 4) {
    int64_t s;
    if (n_iv > 0) {
      if (lo < 0) walk.seek(p);
      s = walk.slot(p);
    } else {
      s = p;
    }
    if (s >= mem_size) break;
    if (lo < 0) {   // lo = first i with sorted_off[i] > s - T ; hi = first i with sorted_off[i] > s
      const int64_t key = s - tile_elems;
      int x = 0, y = ntiles;
      while (x < y) { int mid = (x + y) >> 1; if (sorted_off[mid] > key) y = mid; else x = mid + 1; }
      lo = x;
      y = ntiles;
      while (x < y) { int mid = (x + y) >> 1; if (sorted_off[mid] > s) y = mid; else x = mid + 1; }
      hi = x;
    } else {
      while (lo < ntiles && __ldg(sorted_off + lo) <= s - tile_elems) ++lo;
      if (hi < lo) hi = lo;
      while (hi < ntiles && __ldg(sorted_off + hi) <= s) ++hi;
    }
    if (lo >= hi) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = lo; i < hi; ++i) {
      const int64_t base = int64_t(__ldg(sorted + i)) * tile_elems + (s - __ldg(sorted_off + i));
      for (int sp = 0; sp < nsplit; ++sp) {
        float4 v = *reinterpret_cast<const float4*>(ws + sp * split_stride + base);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    if (s + 4 <= mem_size) {
      float4* d = reinterpret_cast<float4*>(dM + s);
      float4 o = *d;
      o.x += acc.x; o.y += acc.y; o.z += acc.z; o.w += acc.w;
      *d = o;
    } else {   // |M| % 4 != 0: the last group is partial
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
      for (int k = 0; s + k < mem_size; ++k) dM[s + k] += a4[k];
    }
  }
}

// K5 for heavily shared memories (C2 at 100x: ~50 covering tiles x splits per slot): the slab
// kernel below.  NM = 2 reduces two modules' workspaces in one launch: dM = (dM + sum_0) + sum_1.
struct DetMod {
  const float* ws;
  const int32_t* sorted;
  const int64_t* sorted_off;
  const int2* cover;   // static covering range per 4-slot group (built at registration), or null
  int ntiles, nsplit;
};

__device__ __forceinline__ int2 det_cover(const DetMod& m, int64_t s, int64_t tile_elems) {
  if (m.cover) return __ldg(m.cover + (s >> 2));
  int x = 0, y = m.ntiles;
  const int64_t key = s - tile_elems;
  while (x < y) { int mid = (x + y) >> 1; if (__ldg(m.sorted_off + mid) > key) y = mid; else x = mid + 1; }
  const int lo = x;
  y = m.ntiles;
  while (x < y) { int mid = (x + y) >> 1; if (__ldg(m.sorted_off + mid) > s) y = mid; else x = mid + 1; }
  return make_int2(lo, x);
}

template <int NM>
struct DetMods {
  DetMod m[NM];
};

// K5, slab form (heavily shared memories): a CTA takes 32 consecutive slot groups (128 slots,
// lane l = group l) and its NW warps split every module's covering-tile range (the union over the
// 32 groups) into NW contiguous shares.  For each tile of its share a warp reads the partials of
// all 32 groups at once — consecutive 16-B pieces of the same tile, one coalesced 512-B request —
// and each lane adds the terms that cover its group (tiles ascending, splits inner).  The NW
// per-warp sums are combined in warp order through shared memory, then dM += module 0's sum,
// then module 1's: a fixed order, bitwise reproducible.  (The warp-per-group form issues
// scattered 16-B reads, each lane a different tile: 24.6 us at C2 for both modules.)
template <int NM, int NW>
__global__ void __launch_bounds__(NW * 32) det_reduce_slab_kernel(
    float* __restrict__ dM, const __grid_constant__ DetMods<NM> mods, int64_t tile_elems, int64_t mem_size,
    const int64_t* __restrict__ iv_start, const int64_t* __restrict__ iv_prefix, int n_iv, int64_t n_touched) {
  __shared__ float4 part[NM][NW][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n = n_iv > 0 ? n_touched : mem_size;
  const int64_t ngroups = (n + 3) / 4;
  for (int64_t gb = int64_t(blockIdx.x) * 32; gb < ngroups; gb += int64_t(gridDim.x) * 32) {
    const int64_t g = gb + lane;
    int64_t s = g * 4;
    bool valid = g < ngroups;
    if (valid && n_iv > 0) {
      IvWalk iw{iv_start, iv_prefix, n_iv};
      iw.seek(s);
      s = iw.slot(s);
    }
    valid = valid && s < mem_size;
#pragma unroll
    for (int j = 0; j < NM; ++j) {
      const DetMod& m = mods.m[j];
      const int2 r = valid ? det_cover(m, s, tile_elems) : make_int2(0x7fffffff, 0);
      int lo = valid && r.x < r.y ? r.x : 0x7fffffff, hi = valid && r.x < r.y ? r.y : 0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
      }
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lo < hi) {   // warp-uniform
        const int per = (hi - lo + NW - 1) / NW;
        const int a = lo + w * per, b = min(hi, a + per);
        const int64_t split_stride = int64_t(m.ntiles) * tile_elems;
        constexpr int U = 4;
        for (int i0 = a; i0 < b; i0 += U) {
          int t[U];
          int64_t o[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = min(i0 + u, b - 1);
            t[u] = __ldg(m.sorted + i);
            o[u] = __ldg(m.sorted_off + i);
          }
          for (int sp = 0; sp < m.nsplit; ++sp) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int i = i0 + u;
              const bool cov = i < b && i >= r.x && i < r.y && valid;
              v[u] = cov ? *reinterpret_cast<const float4*>(m.ws + sp * split_stride + int64_t(t[u]) * tile_elems + (s - o[u]))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            // order: batches of U tiles ascending, then split, then tile -- fixed by the static
            // covers (the shares and batches do not depend on the data or on timing)
#pragma unroll
            for (int u = 0; u < U; ++u) {
              acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
            }
          }
        }
      }
      part[j][w][lane] = acc;
    }
    __syncthreads();
    if (w == 0 && valid) {
      float4 tot[NM];
#pragma unroll
      for (int j = 0; j < NM; ++j) {
        tot[j] = part[j][0][lane];
#pragma unroll
        for (int k = 1; k < NW; ++k) {
          const float4 p = part[j][k][lane];
          tot[j].x += p.x; tot[j].y += p.y; tot[j].z += p.z; tot[j].w += p.w;
        }
      }
      if (s + 4 <= mem_size) {
        float4* d = reinterpret_cast<float4*>(dM + s);
        float4 o = *d;
#pragma unroll
        for (int j = 0; j < NM; ++j) {
          o.x += tot[j].x; o.y += tot[j].y; o.z += tot[j].z; o.w += tot[j].w;
        }
        *d = o;
      } else {   // |M| % 4 != 0: the last group is partial
        for (int j = 0; j < NM; ++j) {
          const float a4[4] = {tot[j].x, tot[j].y, tot[j].z, tot[j].w};
          for (int k = 0; s + k < mem_size; ++k) dM[s + k] += a4[k];
        }
      }
    }
    __syncthreads();
  }
}

__global__ void sync_shadow_kernel(const float* __restrict__ M, ShadowOut so, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    so.store1(i, __bfloat16_as_ushort(__float2bfloat16_rn(M[i])));
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
  a.neg_base = c->neg_base;
  a.layout = c->cfg.tile_layout;
  return a;
}

int grid_1d(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return int(b < 1 ? 1 : b);
}

// Block tile: 64 x 64 (4 x 4 outputs per thread) unless that leaves most of the 148 SMs idle;
// small problems (C1: 64 tokens x 256) drop to 32 x 32 or 16 x 16 so more CTAs issue the
// dependent hashed gathers in parallel (the 64-tile grid there is 4 CTAs).
int simt_tile(int64_t rows, int64_t cols) {
  for (int ts : {64, 32}) {
    int64_t blocks = ((rows + ts - 1) / ts) * ((cols + ts - 1) / ts);
    if (blocks >= 148) return ts;
  }
  return 16;
}

template <typename XT, typename MT, bool kTransW>
void simt_fwd_ts(int ts, const XT* X, XT* Y, const MT* Mop, const MapArgs& a, int64_t T, int K, int N, float lam,
                 const float* bias, cudaStream_t s) {
  auto grid = [&](int t) { return dim3(unsigned((N + t - 1) / t), unsigned((T + t - 1) / t)); };
  if (ts == 64)
    simt_mm_kernel<XT, MT, kTransW, 64><<<grid(64), 256, 0, s>>>(X, Y, Mop, a, T, K, N, lam, bias);
  else if (ts == 32)
    simt_mm_kernel<XT, MT, kTransW, 32><<<grid(32), 256, 0, s>>>(X, Y, Mop, a, T, K, N, lam, bias);
  else
    simt_mm_kernel<XT, MT, kTransW, 16><<<grid(16), 256, 0, s>>>(X, Y, Mop, a, T, K, N, lam, bias);
}

template <typename XT>
void simt_dw_ts(int ts, const XT* X, const XT* dY, const MapArgs& a, int64_t T, int H, int O, float lam, float* ws,
                float* dM, cudaStream_t s) {
  auto grid = [&](int t) { return dim3(unsigned((O + t - 1) / t), unsigned((H + t - 1) / t)); };
  if (ts == 64)
    simt_dw_kernel<XT, 64><<<grid(64), 256, 0, s>>>(X, dY, a, T, H, O, lam, ws, dM);
  else if (ts == 32)
    simt_dw_kernel<XT, 32><<<grid(32), 256, 0, s>>>(X, dY, a, T, H, O, lam, ws, dM);
  else
    simt_dw_kernel<XT, 16><<<grid(16), 256, 0, s>>>(X, dY, a, T, H, O, lam, ws, dM);
}

}  // namespace

cudaError_t launch_simt_fwd(const Ctx* c, const Module& m, const void* X, void* Y, int64_t T, roast_dtype_t dt,
                            bool transpose_w, cudaStream_t s, const float* bias) {
  if (T == 0) return cudaSuccess;
  const int K = int(transpose_w ? m.O : m.H);
  const int N = int(transpose_w ? m.H : m.O);
  const int ts = simt_tile(T, N);
  MapArgs a = map_args(c, m);
  if (dt == ROAST_FP32) {
    if (transpose_w)
      simt_fwd_ts<float, float, true>(ts, (const float*)X, (float*)Y, c->M, a, T, K, N, m.lam, bias, s);
    else
      simt_fwd_ts<float, float, false>(ts, (const float*)X, (float*)Y, c->M, a, T, K, N, m.lam, bias, s);
  } else {
    auto* sh = reinterpret_cast<const __nv_bfloat16*>(c->shadow);
    if (transpose_w)
      simt_fwd_ts<__nv_bfloat16, __nv_bfloat16, true>(ts, (const __nv_bfloat16*)X, (__nv_bfloat16*)Y, sh, a, T, K, N,
                                                      m.lam, bias, s);
    else
      simt_fwd_ts<__nv_bfloat16, __nv_bfloat16, false>(ts, (const __nv_bfloat16*)X, (__nv_bfloat16*)Y, sh, a, T, K,
                                                       N, m.lam, bias, s);
  }
  return cudaGetLastError();
}

cudaError_t launch_simt_dw(const Ctx* c, const Module& m, const void* X, const void* dY, int64_t T,
                           roast_dtype_t dt, float* ws, cudaStream_t s) {
  const int ts = simt_tile(m.H, m.O);
  MapArgs a = map_args(c, m);
  if (dt == ROAST_FP32)
    simt_dw_ts<float>(ts, (const float*)X, (const float*)dY, a, T, int(m.H), int(m.O), m.lam, ws, c->dM, s);
  else
    simt_dw_ts<__nv_bfloat16>(ts, (const __nv_bfloat16*)X, (const __nv_bfloat16*)dY, a, T, int(m.H), int(m.O),
                              m.lam, ws, c->dM, s);
  return cudaGetLastError();
}

namespace {
// mean number of covering tiles per visited slot: a warp per slot group when it is high (C2 at
// 100x: 50; C5: 1-8, where the per-thread incremental walk wins: 0.72 vs 1.23 ms at 8 MB, 0.75
// vs 4.1 ms at 2 GB)
bool det_warp_variant(const Ctx* c, const Module& m, bool touched) {
  const int64_t visited = touched ? c->touched_n : c->mem_size;
  const double cover = double(int64_t(m.nx) * m.ny) * double(c->tile.z1) * c->tile.z2 / double(std::max<int64_t>(visited, 1));
  return cover >= 16.0;
}

bool det_touched(Ctx* c, cudaStream_t s) {
  if (!(c->touched_valid && c->touched_for == int64_t(c->modules.size()))) {   // build once, eagerly
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) touched_prepare(c, s);
  }
  return c->touched_valid && c->touched_for == int64_t(c->modules.size()) && c->touched_vec && c->n_iv > 0;
}

DetMod det_mod(const Module& m, const float* ws, int nsplit) {
  return DetMod{ws, m.d_sorted, m.d_sorted_off, reinterpret_cast<const int2*>(m.d_cover), m.nx * m.ny, nsplit};
}
}  // namespace

cudaError_t launch_det_reduce2(Ctx* c, const Module& m0, const float* ws0, int ns0, const Module* m1,
                               const float* ws1, int ns1, cudaStream_t s) {
  const bool touched = det_touched(c, s);
  const int threads = 256;
  const int64_t ngroups = ((touched ? c->touched_n : c->mem_size) + 3) / 4;
  const bool warp0 = det_warp_variant(c, m0, touched), warp1 = m1 && det_warp_variant(c, *m1, touched);
  const int64_t* ivs = touched ? c->d_iv : nullptr;
  const int64_t* ivp = touched ? c->d_iv + c->n_iv : nullptr;
  const int niv = touched ? c->n_iv : 0;
  const int64_t nt = touched ? c->touched_n : 0;
  const int64_t te = int64_t(c->tile.z1) * c->tile.z2;
  if (warp0 && (warp1 || !m1)) {
    const int64_t blocks = std::min<int64_t>((ngroups + 31) / 32, 148 * 8);
    if (m1) {
      const DetMods<2> md{{det_mod(m0, ws0, ns0), det_mod(*m1, ws1, ns1)}};
      det_reduce_slab_kernel<2, 8><<<unsigned(blocks), 256, 0, s>>>(c->dM, md, te, c->mem_size, ivs, ivp, niv, nt);
    } else {
      const DetMods<1> md{{det_mod(m0, ws0, ns0)}};
      det_reduce_slab_kernel<1, 8><<<unsigned(blocks), 256, 0, s>>>(c->dM, md, te, c->mem_size, ivs, ivp, niv, nt);
    }
    return cudaGetLastError();
  }
  // per-thread incremental walk, one module per launch (in module order)
  for (int j = 0; j < (m1 ? 2 : 1); ++j) {
    const Module& m = j ? *m1 : m0;
    const int64_t blocks = std::min<int64_t>((ngroups + threads - 1) / threads, 148 * 32);
    det_reduce_kernel<<<unsigned(blocks), threads, 0, s>>>(c->dM, j ? ws1 : ws0, m.d_sorted, m.d_sorted_off,
                                                           m.nx * m.ny, te, j ? ns1 : ns0, c->mem_size, ivs, ivp, niv, nt);
    if (cudaError_t e = cudaGetLastError()) return e;
    if (j) c->launches++;   // the caller counts one launch
  }
  return cudaSuccess;
}

cudaError_t launch_det_reduce(Ctx* c, const Module& m, const float* ws, int nsplit, cudaStream_t s) {
  return launch_det_reduce2(c, m, ws, nsplit, nullptr, nullptr, 0, s);
}

cudaError_t launch_sync_shadow(Ctx* c, cudaStream_t s) {
  sync_shadow_kernel<<<grid_1d(c->mem_size, 256), 256, 0, s>>>(c->M, shadow_out(c), c->mem_size);
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
// One optimizer update of a single slot (fp32 registers in / out).
template <int KIND>
__device__ __forceinline__ float opt_update(float w, float g0, float& a, float& b, float lr, float b1, float b2,
                                            float eps, float wd, float bc1, float bc2) {
  const float g = g0 + wd * w;
  if (KIND == 0) {
    w -= lr * g;
  } else if (KIND == 1) {
    a = a + g * g;
    w -= __fdividef(lr * g, sqrtf(a) + eps);
  } else {
    // bc1 / bc2 arrive as reciprocals of the bias corrections; one fast division per slot keeps
    // the pass HBM-bound (IEEE divisions made it ~70 % issue-bound at 2 GB)
    a = b1 * a + (1.f - b1) * g;
    b = b2 * b + (1.f - b2) * g * g;
    w -= __fdividef(lr * (a * bc1), sqrtf(b * bc2) + eps);
  }
  return w;
}

struct OptArgs {
  float* M;
  float* dM;
  ShadowOut so;
  float* s1;
  float* s2;
  float lr, b1, b2, eps, wd, bc1, bc2;
  int zero;
  // index space: n elements; slot = p (n_iv == 0) or the p-th touched slot (exchange.cu tables)
  int64_t n;
  const float* gpack;   // non-null: the gradient of index p is gpack[p] (the all-reduced packed buffer)
  const int64_t* iv_start;
  const int64_t* iv_prefix;
  int n_iv;
  P2PView p2p;          // world > 0: the gradient of index p is sum_r buf_r[p], read from the peers
};

// NVLS multicast accesses (nvls.cu maps the window's multicast alias): ld_reduce returns the sum
// of every rank's copy of the address, reduced in the NVSwitch; st writes every rank's copy.
__device__ __forceinline__ float4 nvls_ld_reduce4(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ float nvls_ld_reduce1(const float* mc) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ void nvls_st4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
               :: "l"(mc), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void nvls_st1(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" :: "l"(mc), "f"(v) : "memory");
}

// One-shot P2P exchange (p2p.cu): wait until every rank has published this step's packed
// gradient (flags[r] >= epoch, acquire at system scope), then return the buffer parity.  A
// rank that never arrives would hang the GPU, so the wait gives up after 20 s: it sets bit 2 of
// the sticky error word (roast_get_error -> ROAST_ERR_STATE) and traps.
__device__ int p2p_wait(const P2PView& v) {
  __shared__ int s_epoch;
  if (threadIdx.x == 0) {
    const int e = *reinterpret_cast<const volatile int*>(v.epoch);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < v.world; ++r) {
      int f;
      for (;;) {
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(f) : "l"(v.flags + r) : "memory");
        if (f - e >= 0) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {
          atomicOr(v.err, 2);
          __threadfence_system();
          __trap();
        }
        __nanosleep(64);
      }
    }
    s_epoch = e;
  }
  __syncthreads();
  return s_epoch;
}

// One pass over |M| (or over the touched slots): update M from dM (and the optimizer state),
// refresh both halves of the bf16 shadow, optionally zero dM.  kind: 0 SGD, 1 Adagrad, 2 Adam
// (PyTorch formulas).  V = 4: 16-byte vectors (every index-space run is a multiple of 4 and
// 16-byte aligned), V = 1: scalar.
template <int KIND, int V>
__global__ void opt_kernel(OptArgs a) {
  int64_t pbuf = 0;   // P2P: offset of this step's buffer (parity of the epoch)
  if (a.p2p.world > 0) pbuf = (p2p_wait(a.p2p) & 1) ? a.p2p.stride : 0;
  // NVLS: the peers wrote their buffers through unicast mappings; order the multicast reads after
  // the flag acquire across the two address aliases
  if (a.p2p.mc_buf0) asm volatile("fence.proxy.alias;" ::: "memory");
  const int64_t lo = a.p2p.lo, hi = a.p2p.hi < 0 ? a.n : a.p2p.hi;   // two-shot: this rank's slice
  int64_t b, e;
  cta_range(hi - lo, V, &b, &e);
  b += lo;
  e += lo;
  IvWalk walk{a.iv_start, a.iv_prefix, a.n_iv};
  if (a.n_iv > 0 && b + int64_t(threadIdx.x) * V < e) walk.seek(b + int64_t(threadIdx.x) * V);
  for (int64_t p = b + int64_t(threadIdx.x) * V; p < e; p += int64_t(blockDim.x) * V) {
    const int64_t i = a.n_iv == 0 ? p : walk.slot(p);
    float w[V], g[V], x[V], y[V];
    if constexpr (V == 4) {
      const float4 wv = *reinterpret_cast<const float4*>(a.M + i);
      float4 gv;
      if (a.p2p.mc_buf0) {     // NVLS: the sum over the ranks, reduced in the switch
        gv = nvls_ld_reduce4(a.p2p.mc_buf0 + pbuf + p);
      } else if (a.p2p.world > 0) {   // fixed rank order: every rank computes the same sum, so M stays replicated
        gv = __ldcv(reinterpret_cast<const float4*>(a.p2p.buf0[0] + pbuf + p));
        for (int r = 1; r < a.p2p.world; ++r) {
          const float4 v = __ldcv(reinterpret_cast<const float4*>(a.p2p.buf0[r] + pbuf + p));
          gv.x += v.x; gv.y += v.y; gv.z += v.z; gv.w += v.w;
        }
      } else {
        gv = *reinterpret_cast<const float4*>(a.gpack ? a.gpack + p : a.dM + i);
      }
      w[0] = wv.x; w[1] = wv.y; w[2] = wv.z; w[3] = wv.w;
      g[0] = gv.x; g[1] = gv.y; g[2] = gv.z; g[3] = gv.w;
      if (KIND >= 1) {
        const float4 v = *reinterpret_cast<const float4*>(a.s1 + i);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
      }
      if (KIND == 2) {
        const float4 v = *reinterpret_cast<const float4*>(a.s2 + i);
        y[0] = v.x; y[1] = v.y; y[2] = v.z; y[3] = v.w;
      }
    } else {
      w[0] = a.M[i];
      if (a.p2p.mc_buf0) {
        g[0] = nvls_ld_reduce1(a.p2p.mc_buf0 + pbuf + p);
      } else if (a.p2p.world > 0) {
        g[0] = __ldcv(a.p2p.buf0[0] + pbuf + p);
        for (int r = 1; r < a.p2p.world; ++r) g[0] += __ldcv(a.p2p.buf0[r] + pbuf + p);
      } else {
        g[0] = a.gpack ? a.gpack[p] : a.dM[i];
      }
      if (KIND >= 1) x[0] = a.s1[i];
      if (KIND == 2) y[0] = a.s2[i];
    }
#pragma unroll
    for (int k = 0; k < V; ++k) w[k] = opt_update<KIND>(w[k], g[k], x[k], y[k], a.lr, a.b1, a.b2, a.eps, a.wd, a.bc1, a.bc2);
    if (a.p2p.mc_mout) {   // NVLS two-shot: broadcast this slice's new values into every rank's window
      if constexpr (V == 4)
        nvls_st4(a.p2p.mc_mout + p, make_float4(w[0], w[1], w[2], w[3]));
      else
        nvls_st1(a.p2p.mc_mout + p, w[0]);
    } else if (a.p2p.mout) {   // two-shot: publish this slice's new values for the gather phase
      if constexpr (V == 4)
        *reinterpret_cast<float4*>(a.p2p.mout + p) = make_float4(w[0], w[1], w[2], w[3]);
      else
        a.p2p.mout[p] = w[0];
    }
    if constexpr (V == 4) {
      *reinterpret_cast<float4*>(a.M + i) = make_float4(w[0], w[1], w[2], w[3]);
      if (KIND >= 1) *reinterpret_cast<float4*>(a.s1 + i) = make_float4(x[0], x[1], x[2], x[3]);
      if (KIND == 2) *reinterpret_cast<float4*>(a.s2 + i) = make_float4(y[0], y[1], y[2], y[3]);
      const __nv_bfloat162 p0 = __floats2bfloat162_rn(w[0], w[1]), p1 = __floats2bfloat162_rn(w[2], w[3]);
      uint2 pos;
      pos.x = *reinterpret_cast<const uint32_t*>(&p0);
      pos.y = *reinterpret_cast<const uint32_t*>(&p1);
      a.so.store4(i, pos);   // both halves of every replica
      if (a.zero)
        *reinterpret_cast<float4*>(a.dM + i) = make_float4(0.f, 0.f, 0.f, 0.f);
      else if (a.p2p.world > 0)   // keep the documented dM contents: the summed gradient
        *reinterpret_cast<float4*>(a.dM + i) = make_float4(g[0], g[1], g[2], g[3]);
    } else {
      a.M[i] = w[0];
      if (KIND >= 1) a.s1[i] = x[0];
      if (KIND == 2) a.s2[i] = y[0];
      a.so.store1(i, __bfloat16_as_ushort(__float2bfloat16_rn(w[0])));
      if (a.zero)
        a.dM[i] = 0.f;
      else if (a.p2p.world > 0)
        a.dM[i] = g[0];
    }
  }
}

template <int KIND>
void launch_opt_kind(const OptArgs& a, bool vec, cudaStream_t s) {
  const int V = vec ? 4 : 1;
  const int64_t len = a.p2p.hi < 0 ? a.n : a.p2p.hi - a.p2p.lo;
  int64_t blocks = (len / V + 255) / 256;
  blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), 148 * 16);
  if (vec)
    opt_kernel<KIND, 4><<<unsigned(blocks), 256, 0, s>>>(a);
  else
    opt_kernel<KIND, 1><<<unsigned(blocks), 256, 0, s>>>(a);
}

}  // namespace

cudaError_t launch_optimizer(Ctx* c, int kind, float lr, float b1, float b2, float eps, float wd, int64_t step,
                             int zero, bool touched_only, cudaStream_t s, const float* gpack, const P2PView* p2p) {
  OptArgs a{};
  a.gpack = gpack;
  if (p2p) a.p2p = *p2p;
  a.M = c->M;
  a.dM = c->dM;
  a.so = shadow_out(c);
  a.s1 = c->opt_s1;
  a.s2 = c->opt_s2;
  a.lr = lr;
  a.b1 = b1;
  a.b2 = b2;
  a.eps = eps;
  a.wd = wd;
  a.bc1 = kind == 2 ? float(1.0 / (1.0 - pow(double(b1), double(step)))) : 1.f;   // reciprocals
  a.bc2 = kind == 2 ? float(1.0 / (1.0 - pow(double(b2), double(step)))) : 1.f;
  a.zero = zero;
  bool vec;
  if (touched_only) {   // the slots some module can read or write (exchange.cu); the rest are dead
    a.n = c->touched_n;
    a.iv_start = c->d_iv;
    a.iv_prefix = c->d_iv + c->n_iv;
    a.n_iv = c->n_iv;
    vec = c->touched_vec;
    if (a.n == 0) return cudaSuccess;
  } else {
    a.n = c->mem_size;
    vec = c->mem_size % 4 == 0;
  }
  if (kind == 0)
    launch_opt_kind<0>(a, vec, s);
  else if (kind == 1)
    launch_opt_kind<1>(a, vec, s);
  else
    launch_opt_kind<2>(a, vec, s);
  return cudaGetLastError();
}

}  // namespace roast
