// tma_bench.cu — TMA (cp.async.bulk.tensor) L2->smem throughput on one B200, all SMs (standalone).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench.bin tools/tma_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(ph) : "memory");
  } while (!done);
}
__device__ __forceinline__ void load(const CUtensorMap* m, void* dst, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

struct Maps { CUtensorMap a, b; };

// each stage: na boxes from map a (box rows ra) + nb boxes from map b (box rows 64); depth = stages in flight
#ifdef CLUSTER2
#define CLUSTER_ATTR __cluster_dims__(2, 1, 1)
#else
#define CLUSTER_ATTR
#endif
// -DCLUSTER2: the same kernel launched as clusters of 2 CTAs (as the tcgen05 GEMM is)
__global__ void CLUSTER_ATTR k(const __grid_constant__ Maps maps, int iters, int depth, int na, int ra, int nbx, int arows,
                  int brows, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  uint64_t* bars = (uint64_t*)(base + 200 * 1024);
  const int stage_bytes = na * ra * 128 + nbx * 8192;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    long long t0 = clock64();
    uint32_t seed = blockIdx.x * 7919u + 1;
    for (int it = 0; it < iters + depth; ++it) {
      int s = it % depth;
      if (it >= depth) wait(&bars[s], ((it / depth) - 1) & 1);
      if (it < iters) {
        uint8_t* dst = base + s * stage_bytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])),
                     "r"(stage_bytes) : "memory");
        for (int i = 0; i < na; ++i) {
          seed = seed * 1664525u + 1013904223u;
          int row = (seed >> 8) % (arows - ra);
          int col = ((seed >> 4) & 7) * 64 % 768;
          load(&maps.a, dst + i * ra * 128, &bars[s], col, row);
        }
        for (int j = 0; j < nbx; ++j) {
          seed = seed * 1664525u + 1013904223u;
          int row = (seed >> 8) % (brows - 64);
          load(&maps.b, dst + na * ra * 128 + j * 8192, &bars[s], 0, row);
        }
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* f;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)f;
}
static void mk(CUtensorMap* m, void* p, uint64_t cols, uint64_t rows, uint32_t bc, uint32_t br) {
  cuuint64_t d[2] = {cols, rows}, st[1] = {cols * 2};
  cuuint32_t b[2] = {bc, br}, e[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", r);
}

int main() {
  void *A, *B;
  size_t a_rows = 8192, b_rows_small = 1536, b_rows_big = 8192 * 48;
  cudaMalloc(&A, a_rows * 768 * 2);
  cudaMalloc(&B, b_rows_big * 128);
  cudaMemset(A, 0, a_rows * 768 * 2);
  cudaMemset(B, 0, b_rows_big * 128);
  long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Case { const char* name; int na, ra, nbx, depth; size_t brows; int boff = 0; } cases[] = {
      {"A 16KB box{64,128}", 1, 128, 0, 6, b_rows_small},
      {"A 16KB x2 (32KB/stage)", 2, 128, 0, 6, b_rows_small},
      {"B 8KB box{64,64} small-region x4", 0, 128, 4, 6, b_rows_small},
      {"B 8KB big-region x4", 0, 128, 4, 6, b_rows_big},
      {"A16K + B 2x8K small (our CG2)", 1, 128, 2, 6, b_rows_small},
      {"A16K + B 2x8K small depth 4", 1, 128, 2, 4, b_rows_small},
      {"A16K + B 4x8K small (our CG1)", 1, 128, 4, 4, b_rows_small},
      {"A 32KB box{64,256}", 1, 256, 0, 6, b_rows_small},
      {"B 8KB small x4, base +16 B", 0, 128, 4, 6, b_rows_small, 16},
      {"B 8KB small x2 depth 6", 0, 128, 2, 6, b_rows_small},
      {"B 8KB small x2 depth 12", 0, 128, 2, 12, b_rows_small},
      {"A16K + B 2x8K small +16B", 1, 128, 2, 6, b_rows_small, 16},
      {"A32K + B 2x8K small (WM2)", 1, 256, 2, 4, b_rows_small},
  };
  for (auto& c : cases) {
    Maps m;
    mk(&m.a, A, 768, a_rows, 64, c.ra);
    mk(&m.b, (char*)B + c.boff, 64, c.brows - 1, 64, 64);
    int iters = 2000;
    k<<<148, 32, 220 * 1024>>>(m, 10, c.depth, c.na, c.ra, c.nbx, (int)a_rows, (int)c.brows, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 32, 220 * 1024>>>(m, iters, c.depth, c.na, c.ra, c.nbx, (int)a_rows, (int)c.brows, out);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[148];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    double bytes = double(c.na * c.ra * 128 + c.nbx * 8192) * iters;
    printf("%-34s depth %d: %6.1f B/clk/SM  %7.1f GB/s total  (%s)\n", c.name, c.depth, bytes / mx,
           bytes * 148 / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
  }
  return 0;
}
