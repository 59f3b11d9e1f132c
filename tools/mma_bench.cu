// mma_bench.cu — measure tcgen05.mma issue throughput / latency on one B200 (standalone).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_bench tools/mma_bench.cu && /tmp/mma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a),
               "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(ph) : "memory");
  } while (!done);
}

template <int N, int MN_B>
__global__ void k(long long* out, int iters, int commit_every) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  uint64_t* bar = (uint64_t*)(base + 65536);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = *slot;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(MN_B) << 16) | (uint32_t(N >> 3) << 17) | (8u << 24);
  if (threadIdx.x == 0) {
    uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 16384);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = desc(a0 + kk * 32, 16, 1024);
        uint64_t bd = MN_B ? desc(b0 + kk * 2048, 8192, 1024) : desc(b0 + kk * 32, 16, 1024);
        mma(tm + (i & 1) * 256, ad, bd, idesc, 1);
      }
      if (commit_every > 0 && (i % commit_every) == commit_every - 1) {
        commit(bar);
        wait(bar, ph);
        ph ^= 1;
      }
    }
    commit(bar);
    wait(bar, ph);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int MN_B>
void run(const char* name, int grid, int iters, int ce) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * grid);
  auto f = k<N, MN_B>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  f<<<grid, 128, 70000>>>(d, iters, ce);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  f<<<grid, 128, 70000>>>(d, iters, ce);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  double flops = 2.0 * 128 * N * 16 * 4.0 * iters * grid;
  printf("%-28s grid %3d iters %5d commit_every %3d: %8.1f clk/MMA  %7.1f TF (%s)\n", name, grid, iters, ce,
         mx / (4.0 * iters), flops / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<256, 0>("N256 K-major", 1, 2048, 0);
  run<256, 0>("N256 K-major", 148, 2048, 0);
  run<256, 1>("N256 MN-major B", 148, 2048, 0);
  run<128, 0>("N128 K-major", 148, 2048, 0);
  run<256, 0>("N256 commit/wait each kb", 148, 2048, 1);
  run<256, 0>("N256 commit/wait every 4", 148, 2048, 4);
  return 0;
}
