// gemm_sm100.cu — tcgen05 / TMEM / TMA ROAST-MM for sm_100a (K2 fwd, K3 dX, K4 dW->dM).
//
// What is computed (Algorithm 1; backward P:338-346):
//   FWD  Y  = lambda * X  . W~         M = tokens, N = out, K = in
//   DX   dX = lambda * dY . W~^T       M = tokens, N = in,  K = out
//   DW   G  = X^T . dY                 M = in,     N = out, K = tokens
//        dM[h(x,y) + 64 o1 + o2] += lambda * g(x,y) * G[64x + o1, 64y + o2]
// with W~ the signed 64x64 hash tiles of M read through the tile map (a0).
//
// How it maps to B200:
//  * Persistent, warp-specialised: warp 0 issues TMA, warp 1 issues
//    tcgen05.mma (one thread), warp 2 owns TMEM, warps 4..7 drain the
//    accumulator (tcgen05.ld) and run the epilogue.  smem ring with full/empty
//    mbarriers, 2 TMEM accumulators (2 x 256 fp32 columns) so the epilogue of
//    one tile overlaps the MMAs of the next.
//  * CG = 2 (default): a CTA pair (cluster of 2) runs tcgen05.mma.cta_group::2
//    on a 256 x 256 x 16 instruction; each CTA stages its 128 rows of A and
//    half (128 columns) of B, so operand traffic from L2 is 2/3 of the 1-CTA
//    128 x 256 tile and smem operand reads halve.  The leader CTA issues the
//    MMAs; TMA completion bytes of both CTAs land on the leader's barrier;
//    commits multicast to both CTAs.  CG = 1 keeps the 1-SM 128 x 256 tile.
//  * Hashed weight tiles: each 64x64 bf16 tile is 64 rows of 128 B in M.  A
//    2-D TMA box {64, 64} with SWIZZLE_128B lands it in smem as a canonical
//    SW128 operand: MN-major B for FWD (rows = K), and — the same bytes —
//    K-major B for DX (rows = N).  Offsets are only 16-B aligned (A = 8), so
//    the shadow is described by 8 tensor maps, one per 16-byte phase
//    (base + 16 r), each a plain non-overlapping [rows x 128 B] view.
//  * The sign g is folded into the load address: the shadow holds
//    [+bf16(M) | -bf16(M)], and a tile with g = -1 is read from the negated
//    copy (bf16 negation is exact), so no transform pass touches smem.
//  * lambda is applied once in the epilogue (Algorithm 1).
//  * DW: A = X^T and B = dY are both MN-major TMA tiles; the epilogue writes
//    lambda * g * G per hash tile either into a per-tile workspace (reduced
//    in fixed order by K5: deterministic) or with 16-byte vector atomics into
//    dM (fast mode).  Split-K over tokens fills the SMs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <array>
#include <vector>

#include "roast_internal.h"

namespace roast {
namespace sm100 {

constexpr int BM = 128;   // accumulator rows per CTA
constexpr int BN = 256;   // MMA N (columns of the output tile)
constexpr int BK = 64;    // K per pipeline stage (one 128-byte swizzle row of bf16)
constexpr int NUM_THREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr int TMEM_COLS = 512;
constexpr int KB_CHUNK = 64;  // k-blocks whose tile coordinates are staged in smem at a time

// CG: CTAs per MMA (cta_group). WM: M sub-tiles of 128 rows per CTA sharing each B load
// (WM = 2 uses both 256-column TMEM halves for one unit, so the accumulator is single-buffered).
// NU: output columns per unit (MMA N): 256, or 192 (DX, CG = 2, WM = 2 only) for N = 768-wide
// outputs, whose 48 units of 512 x 256 leave 26 of 74 CTA pairs idle (64 units of 512 x 192
// fill one round of 74 with 25 % less work per unit).
template <int CG, int WM, int NU = BN, bool XBUF = false>
struct Cfg {
  static constexpr int A_BYTES = BM * WM * BK * 2;       // this CTA's 128*WM rows of A
  // this CTA's NU/CG columns of B, in whole 64-wide tiles (NU = 192: 96 K-major rows for DX,
  // two MN-major 64-column atoms for FWD)
  static constexpr int B_BYTES = ((NU / CG + 63) / 64) * 64 * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int NBUF = 2;                         // epilogue staging buffers per warp
  // 4 warps x NBUF x (32 rows x 128 B); XBUF (the GELU dX epilogue, 8 RF warps) gives each warp a
  // second 4 KB buffer for the activation input, at the cost of a pipeline stage
  static constexpr int STAGING = (XBUF ? 2 : 1) * 4 * NBUF * 4096;
  static constexpr int FIXED = STAGING + 1024 + 256 + KB_CHUNK * 4 * 4;
  static constexpr int STAGES = (227 * 1024 - FIXED) / STAGE_BYTES > 6 ? 6 : (227 * 1024 - FIXED) / STAGE_BYTES;
  static constexpr int B_SUB = 4 / CG;                   // 64-wide B sub-tiles per CTA
  static constexpr int SMEM = STAGES * STAGE_BYTES + FIXED;
};

enum Mode { FWD = 0, DX = 1, DW = 2 };

// Warp roles.  WM = 2 FWD / DX units fill all 512 TMEM columns, so the accumulator is single-
// buffered and the next unit's MMAs wait for its drain.  There (RF = true) eight epilogue warps
// (two per TMEM lane quadrant, one per M sub-tile) copy the accumulator into registers as packed
// bf16 — 128 x 32-bit per thread — release TMEM, and only then stage and TMA-store the tile while
// the next unit's MMAs run; setmaxnreg moves registers from the producer / MMA warpgroup to them.
template <int MODE, int CG, int WM>
struct Roles {
  static constexpr bool RF = MODE != DW && WM == 2 && CG == 2;
  static constexpr int EPI_WARPS = RF ? 8 : 4;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
};

#ifdef ROAST_DIAG
#define DIAG(p) ((p).exp)
#else
#define DIAG(p) 0
#endif

struct WMaps {
  CUtensorMap m[8];  // shadow viewed from base + 16 r bytes, r = 0..7
};
struct WMapsHalf {
  CUtensorMap m[8];  // the same views with 32-row boxes (half hash tiles, NU = 192)
};

struct Params {
  int64_t T;            // tokens
  int M, N, K;          // GEMM dims in elements (M, N multiples of 64; K ragged only for DW)
  int m_tiles, n_tiles, k_blocks, splits, kb_per_split, units;
  const int64_t* off;   // tile map
  const int8_t* sgn;
  const int32_t* coord; // packed TMA coordinates (FWD: [x][y], DX: [y][x])
  int coord_ld;         // row length of `coord`
  int ny;               // tiles per row of the tile map (out / 64)
  int64_t neg_row;      // row (128 B units) of the negated shadow copy
  int reps, rep_rows;   // shadow replicas (rep_rows rows apart); CTA pair q reads replica q % reps
  float lam;
  __nv_bfloat16* out;   // FWD: Y [T x N], DX: dX [T x N]
  const float* bias;    // FWD only: fp32 [N] added after lambda (recovered by L), or null
  // fused activation (RF epilogue only; the BERT MLP's GELU, an N-op): FWD also writes
  // act_out = act(bf16 Y); DX writes dX = bf16(lambda dY W~^T) * act'(act_in) elementwise
  int act;
  const __nv_bfloat16* act_in;
  __nv_bfloat16* act_out;
  float* dM;            // DW atomic target
  float* ws;            // DW deterministic workspace [splits][ntiles][4096]
  int ntiles;
  long long* prof;      // debug (ROAST_PROF): per-CTA cycle counters, else null
  int epi;              // 0: TMA bulk store / reduce from staging; 1: coalesced st.global / red.global.v4
  int dw3d;             // DW operands loaded as one 3-D TMA box per operand (else 64x64 2-D boxes)
  // diagnostics only (built with -DROAST_DIAG, set by ROAST_EXP; tools/prof_shapes.py; results
  // are garbage): bit 0 skips the epilogue drain, 1 all operand loads, 4 the B loads, 5 the A
  // loads, 6 the output stores.  Compiled out of the product build.
  int exp;
  // chain mode (FWD / DX only; set in the first problem's Params): two GEMMs in one persistent
  // launch, problem 1's A = problem 0's output.  Each pair walks its own static unit list
  // sched[pair * sched_len + i] = prob << 24 | unit (-1 = end), every problem-0 unit before any
  // problem-1 unit (so the waits below cannot deadlock).  flags[u0] counts the epilogue warps
  // whose TMA stores of problem-0 unit u0 are complete; problem 1 loads k-block kb of m-block mb
  // only after flags[mb * n_tiles0 + kb / 4] == 4 * CG.
  int chain;
  const int32_t* sched;
  int sched_len;
  int* flags;
  int* err;             // sticky device error word (chain wait timeout, bit 2)
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// arrive on a barrier given by its shared::cluster address (own or peer CTA)
// Arrive on a barrier given by its shared::cluster address (own or peer CTA).  Used to hand TMEM
// back to the MMA issuer: the data dependency is tcgen05-proxy (ordered by the caller's
// tcgen05.fence::before_thread_sync), so the default .release.cta semantics suffice; a
// .release.cluster arrive made the epilogue wait ~1.7k cycles per unit for its store queue.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
template <int CG>
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, void* dst, uint32_t bar_cluster, int c0, int c1) {
  if (CG == 1)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
        : "memory");
}
template <int CG>
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, void* dst, uint32_t bar_cluster, int c0, int c1,
                                            int c2) {
  if (CG == 1)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
        : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// MMA completion -> arrive on `bar` (CG = 2: on the same barrier in both CTAs of the pair)
template <int CG>
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  if (CG == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  else
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}
template <int CG>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

#define TMEM_LD32(taddr, r)                                                                                       \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%" \
      "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                              \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),           \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),     \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),   \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])    \
      : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version 1 (tcgen05)
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: bf16 x bf16 -> f32, M = 128 * CG, N = n.
__host__ __device__ constexpr uint32_t make_idesc(int a_mn_major, int b_mn_major, int m, int n = BN) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn_major) << 15) | (uint32_t(b_mn_major) << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// spin until *flag >= target (acquire), then order the async proxy (TMA loads) after it.
// After ~4 s (a grid that is not co-resident, e.g. SMs held by another process) it gives up:
// sets bit 2 of the sticky error word (roast_get_error -> ROAST_ERR_STATE, outputs invalid) and
// proceeds, so every CTA still terminates and the context stays usable.
__device__ __forceinline__ void wait_ready(const int* flag, int target, int* err) {
  int v;
  for (uint32_t spins = 0;; ++spins) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    if (spins > (1u << 26)) {
      if (err) atomicOr(err, 4);
      break;
    }
    __nanosleep(64);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void decode_unit(const Params& p, int u, int& mb, int& nb, int& split) {
  split = u / (p.m_tiles * p.n_tiles);
  int r = u - split * p.m_tiles * p.n_tiles;
  mb = r / p.n_tiles;
  nb = r - mb * p.n_tiles;
}

// GELU, tanh form (the original BERT's; torch's gelu(approximate="tanh")), and its derivative
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Folded constants (k0 = sqrt(2 / pi), k1 = 0.044715): with u = x^2, t = tanh(x (k0 + k0 k1 u)),
//   gelu(x)  = h + h t,  h = x / 2
//   gelu'(x) = (1 + t) / 2 + x (1 - t^2) (k0 / 2 + 3 k0 k1 u / 2)
// — the same functions in 5 / 8 fp32 operations + one tanh.approx (the epilogue of a fused
// activation is ALU-bound: 8 warps evaluate it over the whole 256 x 256 tile of each unit).
__device__ __forceinline__ float gelu_tanh(float x) {
  const float u = x * x;
  const float t = tanh_approx(x * fmaf(0.7978845608f * 0.044715f, u, 0.7978845608f));
  const float h = 0.5f * x;
  return fmaf(h, t, h);
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float u = x * x;
  const float t = tanh_approx(x * fmaf(0.7978845608f * 0.044715f, u, 0.7978845608f));
  const float p = fmaf(1.5f * 0.7978845608f * 0.044715f, u, 0.5f * 0.7978845608f);
  const float r = x * fmaf(-t, t, 1.f);
  return fmaf(r, p, fmaf(0.5f, t, 0.5f));
}
// two packed bf16 -> f(a) * g, f(b) * g ... helpers over a packed pair
__device__ __forceinline__ float2 unpack_bf2(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
}
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---------------------------------------------------------------- the kernel
template <int MODE, int CG, int WM, bool CHAIN = false, int NU = BN, bool ACT = false, bool XBUF = false>
__global__ void __launch_bounds__(Roles<MODE, CG, WM>::THREADS, 1)
    roast_mm_sm100(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapOut, const __grid_constant__ WMaps wmaps,
                   const __grid_constant__ Params p0, const __grid_constant__ CUtensorMap mapA1,
                   const __grid_constant__ CUtensorMap mapOut1, const __grid_constant__ Params p1,
                   const __grid_constant__ WMapsHalf hmaps, const __grid_constant__ CUtensorMap mapAct) {
  static_assert(NU == BN || (NU == 192 && MODE != DW && CG == 2 && WM == 2 && !CHAIN), "NU = 192: FWD / DX, 2 x 2");
  static_assert(!XBUF || (ACT && MODE == DX && !CHAIN), "XBUF: the fused-activation dX epilogue");
  using C = Cfg<CG, WM, NU, XBUF>;
  constexpr bool RF = Roles<MODE, CG, WM>::RF;
  constexpr int EPI_WARPS = Roles<MODE, CG, WM>::EPI_WARPS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                        // [STAGES][A_BYTES]
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;               // [STAGES][B_BYTES]
  uint8_t* sStage = smem + C::STAGES * C::STAGE_BYTES;      // epilogue staging [4 warps][2][4 KB] (x2 with XBUF)
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + C::STAGING);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* ubar = reinterpret_cast<uint64_t*>(sStage + C::STAGING + 128);   // [8] ACT DX: U chunk loaded
  int32_t* sCoord = reinterpret_cast<int32_t*>(sStage + C::STAGING + 256);  // [KB_CHUNK * 4]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // programmatic dependent launch: the next GEMM on this stream may be scheduled as soon as
  // every CTA of this grid is resident (it lands on SMs as they free up and runs its prologue
  // under this grid's tail); it waits (griddepcontrol.wait below) before touching global data
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  long long prof_acc[5] = {0, 0, 0, 0, 0};
  long long prof_epi[4] = {0, 0, 0, 0};   // epilogue: TMEM load+wait, staging wait, STS, fence+issue
  const long long t_start = clock64();
  uint64_t g_start = 0;
  if (p0.prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int pair = blockIdx.x / CG;
  const int rrow = p0.reps > 1 ? (pair % p0.reps) * p0.rep_rows : 0;   // this pair's shadow replica
  const int npairs = gridDim.x / CG;
  // i-th unit of this pair: round-robin over one problem, or the pair's chain schedule
  auto unit_at = [&](int i, int& prob, int& u) -> bool {
    if (!CHAIN) {
      prob = 0;
      u = pair + i * npairs;
      return u < p0.units;
    }
    if (i >= p0.sched_len) return false;
    const int code = __ldg(p0.sched + pair * p0.sched_len + i);
    if (code < 0) return false;
    prob = code >> 24;
    u = code & 0xFFFFFF;
    return true;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], RF ? 2 : 1);   // RF: the A and the B producer warp each arrive
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS * CG);
    }
    if constexpr (ACT && MODE == DX)
      for (int w = 0; w < 8; ++w) mbar_init(&ubar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_map(&mapA);
    if (CHAIN) prefetch_map(&mapA1);
    if (MODE == DW) prefetch_map(&mapB);
  }
  if (warp == 2) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  // TMEM base address: re-read from smem where used, so no register stays live across the
  // setmaxnreg role branches
  auto tmem_base_ld = [&]() -> uint32_t { return *reinterpret_cast<volatile uint32_t*>(tmem_slot); };
  // the previous kernel on this stream (launched before us with PDL) has completed and its
  // writes are visible from here on; everything above touched only smem / TMEM / descriptors
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // RF: registers move from warpgroup 0 (producer, MMA, TMEM allocator, idle) to the eight
  // epilogue warps: 128 x 56 + 256 x 224 = 64512 = 384 x 168.  Each role branch executes its own
  // setmaxnreg so ptxas allocates every branch under its own budget.
  if (warp == 0 || (RF && warp == 3)) {
    if constexpr (RF) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    // RF kernels (WM = 2 FWD / DX) split the producer: warp 0 issues the A box (and waits on the
    // chain's ready counters), warp 3 stages the tile coordinates and issues the hashed B tiles;
    // each arrives on the stage's full barrier with its own byte count.  Otherwise warp 0 does both.
    const bool pa = !RF || warp == 0, pb = !RF || warp == 3;
    // ===================== TMA producer (warp 0, both CTAs) =====================
    // Per work unit the whole warp stages the unit's packed tile coordinates
    // (k-blocks x 4, FWD/DX) into smem with coalesced loads; lane 0 then walks
    // the k-blocks and issues this CTA's TMA copies.  The one load latency per
    // unit hides behind the k-blocks already buffered in the ring.
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0;; ++it) {
      int prob, u;
      if (!unit_at(it, prob, u)) break;
      const Params& p = (CHAIN && prob) ? p1 : p0;
      const CUtensorMap* mA = (CHAIN && prob) ? &mapA1 : &mapA;
      int mb, nb, split;
      decode_unit(p, u, mb, nb, split);
      const int kb0 = split * p.kb_per_split;
      const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
      const int n_sub = min(NU / 64, (p.N - nb * NU) / 64);   // valid 64-wide N sub-tiles of the unit
      // this CTA's B sub-tiles: [j0, j1)
      const int j0 = int(rank) * C::B_SUB;
      const int j1 = min(j0 + C::B_SUB, n_sub);
      // DW: valid 64-wide M boxes of this CTA and of the whole pair (for the tx byte count)
      const int row0 = mb * BM * CG * WM + int(rank) * BM * WM;
      const int m_sub = MODE == DW ? max(0, min(2 * WM, (p.M - row0) / 64)) : 0;
      const int m_sub_pair = MODE == DW ? max(0, min(2 * CG * WM, (p.M - mb * BM * CG * WM) / 64)) : 0;
      // bytes landing on the leader's full barrier per stage (both CTAs)
      // DW: one 3-D box per operand per CTA (2*WM 64-wide h blocks of X, 2 o blocks of dY);
      // out-of-range blocks are zero-filled and still counted
      const uint32_t tx_a = MODE == DW ? 0u : uint32_t((DIAG(p) & 32) ? 0 : CG * C::A_BYTES);
      const uint32_t tx_b = MODE == DW ? 0u : uint32_t((DIAG(p) & 16) ? 0 : (MODE == FWD && NU == 192 ? 4 : n_sub) * 64 * 64 * 2);
      const uint32_t tx = MODE == DW ? (p.dw3d ? uint32_t(CG * (C::A_BYTES + C::B_BYTES))
                                               : uint32_t((m_sub_pair + n_sub) * 64 * 64 * 2))
                                     : (RF ? (pa ? tx_a : tx_b) : tx_a + tx_b);
      for (int kc = kb0; kc < kb1; kc += KB_CHUNK) {
        const int kc1 = min(kc + KB_CHUNK, kb1);
        if (MODE != DW && pb) {
          __syncwarp();
          for (int i = lane; i < (kc1 - kc) * 4; i += 32) {
            const int j = i & 3;
            sCoord[i] = j < n_sub ? __ldg(p.coord + int64_t(kc + (i >> 2)) * p.coord_ld + nb * (NU / 64) + j) : 0;
          }
          __syncwarp();
        }
        if (lane == 0) {
          for (int kb = kc; kb < kc1; ++kb) {
            long long tw0 = p.prof ? clock64() : 0;
            mbar_wait(&empty[s], ph ^ 1);
            if (p.prof) prof_acc[0] += clock64() - tw0;
            uint8_t* a = sA + s * C::A_BYTES;
            uint8_t* b = sB + s * C::B_BYTES;
            const uint32_t fb = CG == 2 ? map_to_rank(smem_u32(&full[s]), 0) : smem_u32(&full[s]);
            if (DIAG(p) & 2) {   // diagnostics: MMAs on stale smem, no operand traffic
              if (leader) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
            } else if (leader) mbar_expect_tx(&full[s], tx);
            if (DIAG(p) & 2) {
            } else if (MODE == DW && p.dw3d) {
              tma_load_3d<CG>(mA, a, fb, 0, kb * BK, row0 >> 6);
              tma_load_3d<CG>(&mapB, b, fb, 0, kb * BK, (nb * BN + j0 * 64) >> 6);
            } else if (MODE == DW) {
              for (int i = 0; i < m_sub; ++i) tma_load_2d<CG>(mA, a + i * 8192, fb, row0 + i * 64, kb * BK);
              for (int j = j0; j < j1; ++j)
                tma_load_2d<CG>(&mapB, b + (j - j0) * 8192, fb, nb * BN + j * 64, kb * BK);
            } else {
              // chain: these 64 columns of A are problem 0's output tile (mb, kb / 4)
              if (pa && CHAIN && prob == 1 && (kb & 3) == 0) wait_ready(p0.flags + mb * p0.n_tiles + (kb >> 2), EPI_WARPS * CG, p0.err);
              if (pa && !(DIAG(p) & 32)) tma_load_2d<CG>(mA, a, fb, kb * BK, row0);
              const int32_t* cc = sCoord + (kb - kc) * 4;
              if (!pb) {
              } else if (MODE == FWD && NU == 192 && !(DIAG(p) & 16)) {
                // 96 MN-major B columns per CTA, whole tiles only (a 64-column SW128 atom cannot
                // be half-filled from its right half): rank 0 = tile 0 | tile 1 loaded from its
                // column 32 (its right half lands in the atom's left half, zeros after); rank 1 =
                // tile 2 | tile 1 (left half used).  Accumulator columns [0,64) [64,96) [96,160)
                // [160,192) hold output columns 0-63, 96-127, 128-191, 64-95 (epilogue permutes).
                const int32_t ca = cc[rank ? 2 : 0], cb = cc[1];
                const int ra = (ca >> 4) + ((ca & 8) ? int(p.neg_row) : 0) + rrow;
                const int rb = (cb >> 4) + ((cb & 8) ? int(p.neg_row) : 0) + rrow;
                tma_load_2d<CG>(&wmaps.m[ca & 7], b, fb, 0, ra);
                tma_load_2d<CG>(&wmaps.m[cb & 7], b + 8192, fb, rank ? 0 : 32, rb);
              } else if (NU == 192 && !(DIAG(p) & 16)) {
                // 96 B rows (N) per CTA: rank 0 = tile 0 + rows 0-31 of tile 1, rank 1 = rows
                // 32-63 of tile 1 + tile 2; every piece lands at a 1024-B multiple (SW128 phase)
                const int32_t ca = cc[rank ? 1 : 0], cb = cc[rank ? 2 : 1];
                const int ra = (ca >> 4) + ((ca & 8) ? int(p.neg_row) : 0) + rrow;
                const int rb = (cb >> 4) + ((cb & 8) ? int(p.neg_row) : 0) + rrow;
                if (rank == 0) {
                  tma_load_2d<CG>(&wmaps.m[ca & 7], b, fb, 0, ra);
                  tma_load_2d<CG>(&hmaps.m[cb & 7], b + 8192, fb, 0, rb);
                } else {
                  tma_load_2d<CG>(&hmaps.m[ca & 7], b, fb, 0, ra + 32);
                  tma_load_2d<CG>(&wmaps.m[cb & 7], b + 4096, fb, 0, rb);
                }
              }
              for (int j = j0; j < j1 && pb && NU == BN && !(DIAG(p) & 16); ++j) {
                // FWD: tile (x = kb, y = nb*4 + j); DX: tile (x = nb*4 + j, y = kb).
                // Packed: row << 4 | neg << 3 | phase; negative tiles read the negated shadow.
                const int32_t c = cc[j];
                const int row = (c >> 4) + ((c & 8) ? int(p.neg_row) : 0) + rrow;
                tma_load_2d<CG>(&wmaps.m[c & 7], b + (j - j0) * 8192, fb, 0, row);
              }
            }
            if (++s == C::STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if constexpr (RF) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (lane == 0 && leader) {
      // ===================== MMA issuer (leader CTA, single thread) =====================
      constexpr uint32_t idesc = make_idesc(MODE == DW ? 1 : 0, MODE == FWD || MODE == DW ? 1 : 0, BM * CG, NU);
      // B descriptor strides: MN-major = 64-col sub-tiles 8 KB apart; K-major = 8-row groups 1 KB apart
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;          // WM = 1: double-buffered accumulator index
      uint32_t aph = 0;
      for (int it = 0;; ++it) {
        int prob, u;
        if (!unit_at(it, prob, u)) break;
        const Params& p = (CHAIN && prob) ? p1 : p0;
        int mb, nb, split;
        decode_unit(p, u, mb, nb, split);
        const int kb0 = split * p.kb_per_split;
        const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
        long long tw1 = p.prof ? clock64() : 0;
        mbar_wait(&tempty[acc], aph ^ 1);
        if (p.prof) prof_acc[2] += clock64() - tw1;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base_ld() + uint32_t(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          long long tw2 = p.prof ? clock64() : 0;
          mbar_wait(&full[s], ph);
          if (p.prof) prof_acc[1] += clock64() - tw2;
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t bd;
            if (MODE == FWD || MODE == DW)
              bd = sw128_desc(b0 + k * 2048, 8192, 1024);   // MN-major: LBO = next 64 N, SBO = next 8 K rows
            else
              bd = sw128_desc(b0 + k * 32, 16, 1024);       // K-major view of the same tile bytes (+32 B / K16)
#pragma unroll
            for (int j = 0; j < WM; ++j) {                  // WM M sub-tiles share this B
              const uint32_t aj = a0 + uint32_t(j * BM * 128);
              const uint64_t ad = MODE == DW ? sw128_desc(aj + k * 2048, 8192, 1024)   // MN-major A
                                             : sw128_desc(aj + k * 32, 16, 1024);      // K-major A
              tc_mma<CG>(d_tmem + uint32_t(j * 256), ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          tc_commit<CG>(&empty[s]);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit<CG>(&tfull[acc]);
        if (WM == 1) acc ^= 1;
        if (acc == 0) aph ^= 1;
      }
    }
  } else if (RF && warp < EPI_WARP0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");   // warp 2 (TMEM allocator)
  } else if (RF && warp >= EPI_WARP0) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ===================== epilogue, register-held (WM = 2 FWD / DX) =====================
    // Warp (q, jh) owns accumulator rows q*32 + lane of M sub-tile jh: NU fp32 columns.
    // Phase A: TMEM -> lambda (+ bias) -> packed bf16 in pk[], then release TMEM to the MMA
    // warp.  Phase B: pk[] -> SW128 staging (4 KB, one per warp) -> TMA store, 64 columns at a
    // time, overlapping the next unit's MMAs.
    const int q = warp & 3;
    const int jh = (warp - EPI_WARP0) >> 2;
    uint8_t* buf = sStage + (warp - EPI_WARP0) * 4096;
    // XBUF: this warp's second buffer, where the U chunks land (chunk c + 1 loads while chunk c is
    // computed and stored from `buf`); else U chunks and act(Y) share `buf` with the stores
    uint8_t* buf2 = XBUF ? sStage + 32768 + (warp - EPI_WARP0) * 4096 : buf;
    const uint32_t tempty_leader0 = map_to_rank(smem_u32(&tempty[0]), 0);
    uint32_t aph = 0;
    uint32_t uph = 0;   // ACT DX: parity of this warp's U-chunk barrier
    for (int it = 0;; ++it) {
      int prob, u;
      if (!unit_at(it, prob, u)) break;
      const Params& p = (CHAIN && prob) ? p1 : p0;
      const CUtensorMap* mO = (CHAIN && prob) ? &mapOut1 : &mapOut;
      int mb, nb, split;
      decode_unit(p, u, mb, nb, split);
      const int nsteps = (DIAG(p) & 1) ? 0 : min(NU, p.N - nb * NU) / 64;
      const bool act_u = ACT && (!CHAIN || prob == 0);   // chained: the activation follows problem 0
      if (ACT && MODE == DX && act_u) {   // request U's first chunk now: it lands while the MMAs finish
        const int r0 = mb * BM * CG * WM + int(rank) * BM * WM + jh * BM + q * 32;
        if (lane == 0 && nsteps > 0) {
          // chunks 1.. of this warp's rows into L2 now: their loads below then wait on L2, not HBM
          for (int c = 1; c < nsteps; ++c)
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                             reinterpret_cast<uint64_t>(&mapAct)), "r"(nb * NU + c * 64), "r"(r0)
                         : "memory");
          // XBUF: buf2 was read out by every lane (syncwarp); else wait for the last store's reads
          if (!XBUF) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_expect_tx(&ubar[warp - EPI_WARP0], 4096);
          tma_load_2d<1>(&mapAct, buf2, smem_u32(&ubar[warp - EPI_WARP0]), nb * NU, r0);
        }
      }
      long long tw3 = p.prof ? clock64() : 0;
      mbar_wait(&tfull[0], aph);
      long long tw4 = p.prof ? clock64() : 0;
      if (p.prof) prof_acc[3] += tw4 - tw3;
      tc_fence_after();
      const uint32_t tbase = tmem_base_ld() + uint32_t(jh * 256) + (uint32_t(q * 32) << 16);
      uint32_t pk[NU / 2];
#pragma unroll
      for (int c = 0; c < NU / 64; ++c) {
        if (c < nsteps) {
          uint32_t r[64];
          if (MODE == FWD && NU == 192) {   // output step c from the permuted accumulator columns
            const uint32_t lo = c == 0 ? 0u : c == 1 ? 160u : 96u, hi = c == 0 ? 32u : c == 1 ? 64u : 128u;
            TMEM_LD32(tbase + lo, r);
            TMEM_LD32(tbase + hi, (r + 32));
          } else {
            TMEM_LD32(tbase + uint32_t(c * 64), r);
            TMEM_LD32(tbase + uint32_t(c * 64 + 32), (r + 32));
          }
          tmem_wait_ld();
          if (MODE == FWD && p.bias) {   // Y = bf16(lambda acc + b)
            const float4* b4 = reinterpret_cast<const float4*>(p.bias + nb * NU + c * 64);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float4 bv = __ldg(b4 + i);
              __nv_bfloat162 v0 = __floats2bfloat162_rn(fmaf(p.lam, __uint_as_float(r[4 * i]), bv.x),
                                                        fmaf(p.lam, __uint_as_float(r[4 * i + 1]), bv.y));
              __nv_bfloat162 v1 = __floats2bfloat162_rn(fmaf(p.lam, __uint_as_float(r[4 * i + 2]), bv.z),
                                                        fmaf(p.lam, __uint_as_float(r[4 * i + 3]), bv.w));
              pk[c * 32 + 2 * i] = *reinterpret_cast<uint32_t*>(&v0);
              pk[c * 32 + 2 * i + 1] = *reinterpret_cast<uint32_t*>(&v1);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              __nv_bfloat162 v = __floats2bfloat162_rn(p.lam * __uint_as_float(r[2 * i]),
                                                       p.lam * __uint_as_float(r[2 * i + 1]));
              pk[c * 32 + i] = *reinterpret_cast<uint32_t*>(&v);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0);
      aph ^= 1;
      if (p.prof) prof_epi[0] += clock64() - tw4;
      const int row0 = mb * BM * CG * WM + int(rank) * BM * WM + jh * BM + q * 32;
      // fused activation: this thread's output row (rows past T are neither read nor written)
#pragma unroll
      for (int c = 0; c < NU / 64; ++c) {
        if (c < nsteps) {
          if (ACT && MODE == DX && act_u) {
            // dX = bf16(dh) * act'(U) (or + R): the U chunk (32 rows x 64 columns) arrives by TMA;
            // each thread reads its row into registers.  XBUF: chunk c + 1 is then requested into the
            // second buffer (it lands while this chunk is computed and stored); else chunk c is
            // requested into the staging buffer once the previous store has read it.
            if (!XBUF && lane == 0 && c > 0) {   // chunk 0 was requested before the accumulator wait
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              mbar_expect_tx(&ubar[warp - EPI_WARP0], 4096);
              tma_load_2d<1>(&mapAct, buf, smem_u32(&ubar[warp - EPI_WARP0]), nb * NU + c * 64, row0);
            }
            mbar_wait(&ubar[warp - EPI_WARP0], uph);
            uph ^= 1;
            uint32_t uw_all[32];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const uint32_t a = smem_u32(buf2 + lane * 128 + ((cc ^ (lane & 7)) << 4));
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(uw_all[4 * cc]), "=r"(uw_all[4 * cc + 1]), "=r"(uw_all[4 * cc + 2]),
                             "=r"(uw_all[4 * cc + 3])
                           : "r"(a));
            }
            __syncwarp();   // every row read before the buffer is reused
            if (XBUF && lane == 0 && c + 1 < nsteps) {
              mbar_expect_tx(&ubar[warp - EPI_WARP0], 4096);
              tma_load_2d<1>(&mapAct, buf2, smem_u32(&ubar[warp - EPI_WARP0]), nb * NU + (c + 1) * 64, row0);
            }
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const uint32_t* uw = uw_all + 4 * cc;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 d = unpack_bf2(pk[c * 32 + 4 * cc + e]), x = unpack_bf2(uw[e]);
                // act 2 (residual): dX = bf16(bf16(dh) + R), the bits of a separate bf16 add
                pk[c * 32 + 4 * cc + e] = p.act == 2 ? pack_bf2(d.x + x.x, d.y + x.y)
                                                     : pack_bf2(d.x * gelu_tanh_grad(x.x), d.y * gelu_tanh_grad(x.y));
              }
            }
          }
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const uint32_t a = smem_u32(buf + lane * 128 + ((cc ^ (lane & 7)) << 4));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pk[c * 32 + 4 * cc]),
                         "r"(pk[c * 32 + 4 * cc + 1]), "r"(pk[c * 32 + 4 * cc + 2]), "r"(pk[c * 32 + 4 * cc + 3])
                         : "memory");
          }
          uint32_t gk[ACT && MODE == FWD ? 32 : 1];   // FWD: act(bf16 Y) of this chunk, staged after Y
          if (ACT && MODE == FWD && act_u) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float2 x = unpack_bf2(pk[c * 32 + i]);
              gk[i] = pack_bf2(gelu_tanh(x.x), gelu_tanh(x.y));
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && !(DIAG(p) & 64)) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(mO)),
                         "r"(nb * NU + c * 64), "r"(row0), "r"(smem_u32(buf))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          if (ACT && MODE == FWD && act_u) {   // the act output through the same staging buffer (mapAct)
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const uint32_t a = smem_u32(buf2 + lane * 128 + ((cc ^ (lane & 7)) << 4));
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(gk[4 * cc]), "r"(gk[4 * cc + 1]),
                           "r"(gk[4 * cc + 2]), "r"(gk[4 * cc + 3])
                           : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                               reinterpret_cast<uint64_t>(&mapAct)),
                           "r"(nb * NU + c * 64), "r"(row0), "r"(smem_u32(buf2))
                           : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          }
        }
      }
      if (p.prof) prof_acc[4] += clock64() - tw4;
      if (CHAIN && prob == 0) {
        // publish this warp's 32 rows of the problem-0 tile: writes complete, then release
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p0.flags + u) : "memory");
        }
        __syncwarp();
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  } else if (!RF && warp >= EPI_WARP0) {
    // ===================== epilogue: TMEM -> registers -> global =====================
    const int q = warp & 3;          // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;   // accumulator row owned by this thread
    const uint32_t tempty_leader0 = CG == 2 ? map_to_rank(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
    int stg = 0;   // staging buffer counter (double buffer per warp)
    int acc = 0;
    uint32_t aph = 0;
    for (int it = 0;; ++it) {
      int prob, u;
      if (!unit_at(it, prob, u)) break;
      const Params& p = (CHAIN && prob) ? p1 : p0;
      const CUtensorMap* mO = (CHAIN && prob) ? &mapOut1 : &mapOut;
      int mb, nb, split;
      decode_unit(p, u, mb, nb, split);
      const int n_valid = min(NU, p.N - nb * NU);
      // DW: each warp's 32 rows of sub-tile j lie in one hash-tile row x; lanes 0..3
      // fetch the (offset, lambda*g) of tiles (x, 4 nb + lane) before the accumulator wait.
      int64_t t_off[WM];
      float t_scale[WM];
#pragma unroll
      for (int j = 0; j < WM; ++j) {
        t_off[j] = 0;
        t_scale[j] = 0.f;
        const int rb = mb * BM * CG * WM + int(rank) * BM * WM + j * BM + q * 32;
        const int y = nb * 4 + (lane & 3);
        if (MODE == DW && lane < 4 && rb < p.M && y * 64 < p.N) {
          const int t = (rb >> 6) * p.ny + y;
          t_off[j] = p.ws ? (int64_t(split) * p.ntiles + t) * 4096 : p.off[t];
          t_scale[j] = p.sgn[t] < 0 ? -p.lam : p.lam;
        }
      }
      long long tw3 = p.prof ? clock64() : 0;
      mbar_wait(&tfull[acc], aph);
      long long tw4 = p.prof ? clock64() : 0;
      if (p.prof) prof_acc[3] += tw4 - tw3;
      tc_fence_after();
#pragma unroll 1
      for (int j = 0; j < WM; ++j) {
        const int row_base = mb * BM * CG * WM + int(rank) * BM * WM + j * BM;
        const uint32_t tbase = tmem_base_ld() + uint32_t(acc * BN + j * 256) + (uint32_t(q * 32) << 16);
        // Each step drains 32 rows x 128 B of output through a 4 KB SW128-swizzled
        // staging buffer (conflict-free st.shared) and one TMA bulk tensor op:
        // FWD/DX store 64 bf16 columns of Y / dX; DW stores (deterministic
        // workspace) or reduce-adds in L2 (dM) 32 fp32 columns of one hash tile.
        constexpr int COLS = MODE == DW ? 32 : 64;
        const int nsteps = n_valid / COLS;
        auto tload = [&](int c, uint32_t (&r)[64]) {
          if (MODE == FWD && NU == 192) {   // output step c from the permuted accumulator columns
            const uint32_t lo = c == 0 ? 0u : c == 1 ? 160u : 96u, hi = c == 0 ? 32u : c == 1 ? 64u : 128u;
            TMEM_LD32(tbase + lo, r);
            TMEM_LD32(tbase + hi, (r + 32));
          } else if (MODE != DW) {
            TMEM_LD32(tbase + uint32_t(c * 64), r);
            TMEM_LD32(tbase + uint32_t(c * 64 + 32), (r + 32));
          } else {
            TMEM_LD32(tbase + uint32_t(c * 32), r);
          }
        };
        auto process = [&](int c, uint32_t (&r)[64]) {
          uint32_t pk[32];
          int64_t tb = 0;
          if (MODE == FWD && p.bias) {
            // Y = bf16(lambda acc + b): the 64 columns' bias, broadcast to every lane from L1
            const float4* b4 = reinterpret_cast<const float4*>(p.bias + nb * NU + c * 64);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float4 bv = __ldg(b4 + i);
              __nv_bfloat162 v0 = __floats2bfloat162_rn(fmaf(p.lam, __uint_as_float(r[4 * i]), bv.x),
                                                        fmaf(p.lam, __uint_as_float(r[4 * i + 1]), bv.y));
              __nv_bfloat162 v1 = __floats2bfloat162_rn(fmaf(p.lam, __uint_as_float(r[4 * i + 2]), bv.z),
                                                        fmaf(p.lam, __uint_as_float(r[4 * i + 3]), bv.w));
              pk[2 * i] = *reinterpret_cast<uint32_t*>(&v0);
              pk[2 * i + 1] = *reinterpret_cast<uint32_t*>(&v1);
            }
          } else if (MODE != DW) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              __nv_bfloat162 v = __floats2bfloat162_rn(p.lam * __uint_as_float(r[2 * i]),
                                                       p.lam * __uint_as_float(r[2 * i + 1]));
              pk[i] = *reinterpret_cast<uint32_t*>(&v);
            }
          } else {
            const float scale = __shfl_sync(0xffffffffu, t_scale[j], c >> 1);
            tb = __shfl_sync(0xffffffffu, t_off[j], c >> 1);
#pragma unroll
            for (int i = 0; i < 32; ++i) pk[i] = __float_as_uint(scale * __uint_as_float(r[i]));
          }
          uint8_t* buf = sStage + (warp - EPI_WARP0) * (C::NBUF * 4096) + (stg % C::NBUF) * 4096;
          long long e1 = p.prof ? clock64() : 0;
          if (lane == 0 && p.epi == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          long long e2 = p.prof ? clock64() : 0;
          if (p.prof) prof_epi[1] += e2 - e1;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const uint32_t a = smem_u32(buf + lane * 128 + ((cc ^ (lane & 7)) << 4));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pk[4 * cc]), "r"(pk[4 * cc + 1]),
                         "r"(pk[4 * cc + 2]), "r"(pk[4 * cc + 3])
                         : "memory");
          }
          if (p.epi == 1) {
            // transpose through the staging buffer: each warp store covers 4 full 128-B rows
            __syncwarp();
            const int rb = row_base + q * 32;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int idx = i * 32 + lane, rr = idx >> 3, ch = idx & 7;
              uint4 v;
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                           : "r"(smem_u32(buf + rr * 128 + ((ch ^ (rr & 7)) << 4))));
              if (MODE != DW) {
                const int64_t m = int64_t(rb) + rr;
                if (m < p.T) *reinterpret_cast<uint4*>(p.out + m * p.N + nb * NU + c * 64 + ch * 8) = v;
              } else if (rb < p.M) {
                float* dst = (p.ws ? p.ws : p.dM) + tb + ((rb + rr) & 63) * 64 + (c & 1) * 32 + ch * 4;
                const float4 f = make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z),
                                             __uint_as_float(v.w));
                if (p.ws)
                  *reinterpret_cast<float4*>(dst) = f;
                else
                  atomicAdd(reinterpret_cast<float4*>(dst), f);
              }
            }
            ++stg;
            return;
          }
          long long e3 = p.prof ? clock64() : 0;
          if (p.prof) prof_epi[2] += e3 - e2;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (p.prof) prof_epi[3] += clock64() - e3;
          if (lane == 0 && !(DIAG(p) & 64)) {
            const uint32_t sb = smem_u32(buf);
            if (MODE != DW) {
              const int x0 = nb * NU + c * 64, y0 = row_base + q * 32;
              asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                               reinterpret_cast<uint64_t>(mO)),
                           "r"(x0), "r"(y0), "r"(sb)
                           : "memory");
            } else if (row_base + q * 32 < p.M) {   // warps past the last hash-tile row write nothing
              const int x0 = (c & 1) * 32;
              const int y0 = int(tb >> 6) + ((row_base + q * 32) & 63);
              if (p.ws)   // deterministic: plain store into the per-tile workspace [.. x 64] fp32
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                 reinterpret_cast<uint64_t>(mO)),
                             "r"(x0), "r"(y0), "r"(sb)
                             : "memory");
              else        // fast: TMA reduce-add into dM in L2 through the 32-byte-phase view of dM
                asm volatile(
                    "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                        reinterpret_cast<uint64_t>(&wmaps.m[(tb >> 3) & 7])),
                    "r"(x0), "r"(y0), "r"(sb)
                    : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++stg;
        };
        uint32_t ra[64];
        for (int c = 0; c < ((DIAG(p) & 1) ? 0 : nsteps); ++c) {
          long long e0 = p.prof ? clock64() : 0;
          tload(c, ra);
          tmem_wait_ld();
          if (p.prof) prof_epi[0] += clock64() - e0;
          process(c, ra);
        }
      }
      if (p.prof) prof_acc[4] += clock64() - tw4;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + uint32_t(acc * 8));
      if (CHAIN && prob == 0) {
        // publish this warp's 32 rows of the problem-0 tile: writes complete, then release
        if (lane == 0) {
          asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p0.flags + u) : "memory");
        }
        __syncwarp();
      }
      if (WM == 1) acc ^= 1;
      if (acc == 0) aph ^= 1;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // staging reads + writes done
    __syncwarp();
  }

  if (p0.prof && lane == 0) {
    long long* o = p0.prof + blockIdx.x * 8;
    if (warp == 0) {
      o[5] = clock64() - t_start;
      uint64_t g_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
      o[3] = (long long)(g_end - g_start);   // ns
    }
    if (warp == 1) { o[1] = prof_acc[1]; if (RF) o[0] = prof_acc[2]; }   // RF: slot 0 = MMA wait for TMEM
    if (warp == EPI_WARP0) { o[4] = prof_acc[4]; o[6] = prof_epi[0]; o[7] = prof_epi[1]; o[2] = prof_epi[2]; if (!RF) o[0] = prof_epi[3]; }
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_ld()), "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_ld()), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- fused backward (MIX)
// The whole backward of a chained layer pair a -> b (Y_a = X_a W_a, Y_b = Y_a W_b) in ONE
// persistent launch, its four GEMMs co-scheduled on the 74 CTA pairs (Alg. 1):
//   P0  DX  dY_a = lambda_b dY_b W~_b^T               (WM = 2, register-held epilogue)
//   P1  DW  dM  += scatter_b(lambda_b g  Y_a^T dY_b)  (WM = 1, split-K, TMA reduce-add)
//   P2  DX  dX_a = lambda_a dY_a W~_a^T               (A = P0's output: waits on P0's tiles)
//   P3  DW  dM  += scatter_a(lambda_a g  X_a^T dY_a)  (B = P0's output: waits on P0's tiles)
// Alone, each GEMM is quantised on its own unit grid (C2: 192 / 72 / 48 / 72 units for 74
// pairs) and the two-stream overlap of separate launches is left to the hardware.  Here every
// pair walks a static unit list from a list-scheduling simulation (host, plan_mix): P0's units
// first on every pair (so no wait can deadlock: all pairs are co-resident, checked at plan
// time), P1 units as filler, P2 / P3 units as soon as the P0 tiles they read are published.
// TMEM is split into two 256-column halves with their own full / empty barriers: a DX unit
// (512 x 256 per pair) takes both, a DW unit (256 x 256) one, alternating, so DW units are
// double-buffered and DX units drain into registers before their stores.
struct MixProb {
  int mode;                 // DX or DW
  int M, N, K;              // GEMM dims (DX: M = tokens; DW: M = in_features, K = tokens)
  int m_tiles, n_tiles, k_blocks, kb_per_split, units;
  const int32_t* coord;     // DX: packed hash-tile TMA coordinates [y][x] (K-major B)
  int coord_ld;
  const int64_t* off;       // DW: tile offsets / signs [x][y]
  const int8_t* sgn;
  int ny;
  float lam;
  int dep;                  // problem whose output tiles this one reads (0) or -1
  int publish;              // 1: this problem's units publish ready counters (P0)
  int ws_slot;              // DW, deterministic: index of its workspace map (maps.ws), else -1
  int act;                  // DX: multiply the output by act'(U) (U from maps.u; the BERT MLP's GELU)
  int ntiles;               // DW: hash tiles of the module (workspace row = (split * ntiles + t) * 64)
};
struct MixParams {
  MixProb p[4];
  int64_t neg_row;          // row (128 B) of the negated shadow copy
  int reps, rep_rows;       // shadow replicas (rep_rows rows apart); CTA pair q reads replica q % reps
  int dm_reps, dm_rep_rows; // dM replicas (fast mode, tiny |M|): CTA pair q reduce-adds into replica q % dm_reps
  const int32_t* sched;     // [pairs][sched_len] codes prob << 24 | unit, -1 = end
  int sched_len;
  int* flags;               // ready counters of the publishing problem's units
  int dep_n_tiles;          // n_tiles of the publishing problem (flag index = mb * this + nb)
  int dep_m_tiles;          // ... and its m_tiles
  int* err;                 // sticky device error word
  long long* prof;
  int exp;                  // diagnostics only (ROAST_EXP in a ROAST_DIAG build): bit 0 no conversion math, bit 1 no TMEM loads
};
struct MixMaps {
  CUtensorMap a[4];         // DX: A (tokens x K); DW: X blocks (3-D)
  CUtensorMap b[4];         // DX: output (tokens x N); DW: dY blocks (3-D)
  WMaps shadow;             // bf16 shadow, 8 phase views (DX B tiles)
  WMaps dm;                 // dM, 8 fp32 phase views (DW reduce-add)
  CUtensorMap ws[2];        // deterministic mode: per-tile fp32 workspaces of the two DW problems
  CUtensorMap u;            // act: the pre-activation U [tokens x N] bf16, 32 x 64 boxes
};

constexpr int MIX_THREADS = 384;
constexpr int MIX_STAGES = 4;
constexpr int MIX_A = 32768, MIX_B = 16384;          // per-stage A / B slots of a DX k-block (32 + 16 KB)
constexpr int MIX_STAGE = MIX_A + MIX_B;              // one stage: [A | B], 48 KB contiguous
// A DW k-block spans MIX_DWBK tokens so that it fills a whole 48 KB stage too (X^T and dY boxes of
// 2 x 64 columns x 96 tokens, 24 KB each): 50 % more weight-gradient operand bytes in flight than
// 64-token blocks (16 + 16 KB of each 48 KB stage); the fused backward is latency-sensitive
// (4 -> 3 stages: 120.8 -> 137.2 us)
constexpr int MIX_DWBK = 96;
constexpr int MIX_DW_BOX = 2 * MIX_DWBK * 128;        // bytes of one DW operand box (2 blocks of 64 columns)
constexpr int MIX_SMEM = MIX_STAGES * (MIX_A + MIX_B) + 8 * 4096 + 1024 + 256 + KB_CHUNK * 4 * 4;

__device__ __forceinline__ void mbar_arrive_cluster_n(uint32_t cluster_addr, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr), "r"(n)
               : "memory");
}

__device__ __forceinline__ void mix_decode(const MixProb& P, int u, int& mb, int& nb, int& split) {
  split = u / (P.m_tiles * P.n_tiles);
  const int r = u - split * P.m_tiles * P.n_tiles;
  mb = r / P.n_tiles;
  nb = r - mb * P.n_tiles;
}

__global__ void __launch_bounds__(MIX_THREADS, 1)
    roast_mix_sm100(const __grid_constant__ MixMaps maps, const __grid_constant__ MixParams mp) {
  constexpr int CG = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s = [A 32 KB | B 16 KB] at smem + s * MIX_STAGE (DW: [X^T 24 KB | dY 24 KB])
  auto sA = [&](int st) { return smem + st * MIX_STAGE; };
  auto sB = [&](int st) { return smem + st * MIX_STAGE + MIX_A; };
  uint8_t* sStage = smem + MIX_STAGES * (MIX_A + MIX_B);        // [8 warps][4 KB]
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 8 * 4096);
  uint64_t* empty = full + MIX_STAGES;
  uint64_t* tfull = empty + MIX_STAGES;                         // per TMEM half
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* ubar = reinterpret_cast<uint64_t*>(sStage + 8 * 4096 + 128);   // [8] act: U chunk loaded
  int32_t* sCoord = reinterpret_cast<int32_t*>(sStage + 8 * 4096 + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x / CG;
  const int rrow = mp.reps > 1 ? (pair % mp.reps) * mp.rep_rows : 0;   // this pair's shadow replica
  const int drow = mp.dm_reps > 1 ? (pair % mp.dm_reps) * mp.dm_rep_rows : 0;   // ... and dM replica
  auto unit_at = [&](int i, int& prob, int& u) -> bool {
    if (i >= mp.sched_len) return false;
    const int code = __ldg(mp.sched + pair * mp.sched_len + i);
    if (code < 0) return false;
    prob = code >> 24;
    u = code & 0xFFFFFF;
    return true;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < MIX_STAGES; ++s) {
      mbar_init(&full[s], 2);          // the A and the B producer each arrive (with their tx bytes)
      mbar_init(&empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 1);
      mbar_init(&tempty[h], 8 * CG);   // DW: 8 warps x 1; DX: the half's 4 warps x 2
    }
    for (int w = 0; w < 8; ++w) mbar_init(&ubar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 4; ++i) {
      prefetch_map(&maps.a[i]);
      prefetch_map(&maps.b[i]);
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  auto tmem_base_ld = [&]() -> uint32_t { return *reinterpret_cast<volatile uint32_t*>(tmem_slot); };
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const long long t_start = clock64();
  // ROAST_PROF counters: producer dependency waits; MMA issuer waits for stage data / TMEM (DX, DW)
  long long pw_dep = 0, mw_full = 0, mw_tmem = 0, mw_full_dw = 0, mw_tmem_dw = 0, ep_a = 0, ep_b = 0, ep_n = 0;
  if (warp == 0 || warp == 3) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    // ===================== TMA producers =====================
    // warp 0 loads the A operand, warp 3 the B operand of every stage (each arrives on the
    // stage's full barrier with its own byte count): two issuing threads keep the small-box
    // TMA stream ahead of the MMAs.  The one whose operand is a dependency's output waits for
    // the published tiles: A for DX (dY_a), B for DW (dY_a).
    const bool pa = warp == 0;
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0;; ++it) {
      int prob, u;
      if (!unit_at(it, prob, u)) break;
      const MixProb& P = mp.p[prob];
      int mb, nb, split;
      mix_decode(P, u, mb, nb, split);
      const int kb0 = split * P.kb_per_split;
      const int kb1 = min(kb0 + P.kb_per_split, P.k_blocks);
      if (P.mode == DX) {
        const int row0 = mb * 512 + int(rank) * 256;
        const uint32_t tx = pa ? uint32_t(CG * MIX_A) : uint32_t(4 * 8192);
        for (int kc = kb0; kc < kb1; kc += KB_CHUNK) {
          const int kc1 = min(kc + KB_CHUNK, kb1);
          if (!pa) {
            __syncwarp();
            for (int i = lane; i < (kc1 - kc) * 4; i += 32)
              sCoord[i] = __ldg(P.coord + int64_t(kc + (i >> 2)) * P.coord_ld + nb * 4 + (i & 3));
            __syncwarp();
          }
          if (lane == 0) {
            for (int kb = kc; kb < kc1; ++kb) {
              mbar_wait(&empty[s], ph ^ 1);
              const uint32_t fb = map_to_rank(smem_u32(&full[s]), 0);
              if (leader) mbar_expect_tx(&full[s], tx);
              if (pa) {
                // A = the dependency's output tile (mb, kb / 4) once it is published
                if (P.dep >= 0 && (kb & 3) == 0) {
                  const long long t0 = mp.prof ? clock64() : 0;
                  wait_ready(mp.flags + mb * mp.dep_n_tiles + (kb >> 2), 8 * CG, mp.err);
                  if (mp.prof) pw_dep += clock64() - t0;
                }
                tma_load_2d<CG>(&maps.a[prob], sA(s), fb, kb * BK, row0);
              } else {
                const int32_t* cc = sCoord + (kb - kc) * 4;
                for (int j = 0; j < 2; ++j) {   // this CTA's two 64-row K-major B tiles (x = nb*4 + 2 rank + j, y = kb)
                  const int32_t c = cc[int(rank) * 2 + j];
                  const int row = (c >> 4) + ((c & 8) ? int(mp.neg_row) : 0) + rrow;
                  tma_load_2d<CG>(&maps.shadow.m[c & 7], sB(s) + j * 8192, fb, 0, row);
                }
              }
              if (++s == MIX_STAGES) {
                s = 0;
                ph ^= 1;
              }
            }
          }
        }
      } else {   // DW: X^T and dY as 3-D MN-major boxes (2 x 64-wide blocks x MIX_DWBK tokens per CTA)
        const int row0 = mb * 256 + int(rank) * 128;
        const int col0 = nb * 256 + int(rank) * 128;
        const uint32_t tx = uint32_t(CG * MIX_DW_BOX);
        int waited = -1;   // B producer: last m-block of the dependency waited for in this unit
        if (lane == 0) {
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            const uint32_t fb = map_to_rank(smem_u32(&full[s]), 0);
            if (leader) mbar_expect_tx(&full[s], tx);
            if (pa) {
              tma_load_3d<CG>(&maps.a[prob], sA(s), fb, 0, kb * MIX_DWBK, row0 >> 6);
            } else {
              // B = the dependency's output rows kb*MIX_DWBK.. (512-row m-blocks), columns of tile nb
              if (P.dep >= 0) {
                const int mlast = min((kb * MIX_DWBK + MIX_DWBK - 1) >> 9, mp.dep_m_tiles - 1);
                for (int mbk = max((kb * MIX_DWBK) >> 9, waited + 1); mbk <= mlast; ++mbk) {
                  const long long t0 = mp.prof ? clock64() : 0;
                  wait_ready(mp.flags + mbk * mp.dep_n_tiles + nb, 8 * CG, mp.err);
                  if (mp.prof) pw_dep += clock64() - t0;
                  waited = mbk;
                }
              }
              tma_load_3d<CG>(&maps.b[prob], sA(s) + MIX_DW_BOX, fb, 0, kb * MIX_DWBK, col0 >> 6);
            }
            if (++s == MIX_STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (lane == 0 && leader) {
      // ===================== MMA issuer (leader CTA, one thread) =====================
      constexpr uint32_t idesc_dx = make_idesc(0, 0, 256, 256);
      constexpr uint32_t idesc_dw = make_idesc(1, 1, 256, 256);
      int s = 0;
      uint32_t ph = 0;
      uint32_t usep = 0;          // bit h: parity of the number of uses of TMEM half h so far
      int dwh = 0;                // TMEM half of the next DW unit (alternates)
      for (int it = 0;; ++it) {
        int prob, u;
        if (!unit_at(it, prob, u)) break;
        const MixProb& P = mp.p[prob];
        int mb, nb, split;
        mix_decode(P, u, mb, nb, split);
        const int kb0 = split * P.kb_per_split;
        const int kb1 = min(kb0 + P.kb_per_split, P.k_blocks);
        const uint32_t tbase = tmem_base_ld();
        if (P.mode == DX) {
          long long t0 = mp.prof ? clock64() : 0;
          mbar_wait(&tempty[0], (usep & 1) ^ 1);
          mbar_wait(&tempty[1], ((usep >> 1) & 1) ^ 1);
          if (mp.prof) mw_tmem += clock64() - t0;
          tc_fence_after();
          for (int kb = kb0; kb < kb1; ++kb) {
            t0 = mp.prof ? clock64() : 0;
            mbar_wait(&full[s], ph);
            if (mp.prof) mw_full += clock64() - t0;
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA(s));
            const uint32_t b0 = smem_u32(sB(s));
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t bd = sw128_desc(b0 + k * 32, 16, 1024);   // K-major B
#pragma unroll
              for (int j = 0; j < 2; ++j)
                tc_mma<CG>(tbase + uint32_t(j * 256), sw128_desc(a0 + uint32_t(j * BM * 128) + k * 32, 16, 1024), bd,
                           idesc_dx, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            tc_commit<CG>(&empty[s]);
            if (++s == MIX_STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
          tc_commit<CG>(&tfull[0]);
          tc_commit<CG>(&tfull[1]);
          usep ^= 3u;
        } else {
          const int h = dwh;
          dwh ^= 1;
          long long t0 = mp.prof ? clock64() : 0;
          mbar_wait(&tempty[h], ((usep >> h) & 1) ^ 1);
          if (mp.prof) mw_tmem_dw += clock64() - t0;
          tc_fence_after();
          const uint32_t d = tbase + uint32_t(h * 256);
          for (int kb = kb0; kb < kb1; ++kb) {
            t0 = mp.prof ? clock64() : 0;
            mbar_wait(&full[s], ph);
            if (mp.prof) mw_full_dw += clock64() - t0;
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA(s));
            const uint32_t b0 = a0 + MIX_DW_BOX;
            // MN-major operands: LBO = the next 64-column block (MIX_DWBK rows of 128 B), SBO = the
            // next 8 token rows
#pragma unroll
            for (int k = 0; k < MIX_DWBK / 16; ++k)
              tc_mma<CG>(d, sw128_desc(a0 + k * 2048, MIX_DWBK * 128, 1024),
                         sw128_desc(b0 + k * 2048, MIX_DWBK * 128, 1024), idesc_dw, (kb > kb0 || k > 0) ? 1u : 0u);
            tc_commit<CG>(&empty[s]);
            if (++s == MIX_STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
          tc_commit<CG>(&tfull[h]);
          usep ^= 1u << h;
        }
      }
    }
  } else if (warp < EPI_WARP0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");   // warp 2 (TMEM allocator)
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ===================== epilogue (8 warps) =====================
    const int q = warp & 3;                  // TMEM lane quadrant
    const int jh = (warp - EPI_WARP0) >> 2;  // DX: M sub-tile (= TMEM half); DW: column half
    uint8_t* buf = sStage + (warp - EPI_WARP0) * 4096;
    const uint32_t tempty_leader0 = map_to_rank(smem_u32(&tempty[0]), 0);
    uint32_t usep = 0;   // bit h: parity of the uses of TMEM half h so far (as the MMA issuer's)
    int dwh = 0;
    uint32_t uph = 0;    // act: parity of this warp's U-chunk barrier
    for (int it = 0;; ++it) {
      int prob, u;
      if (!unit_at(it, prob, u)) break;
      const MixProb& P = mp.p[prob];
      int mb, nb, split;
      mix_decode(P, u, mb, nb, split);
      if (P.mode == DX) {
        mbar_wait(&tfull[jh], (usep >> jh) & 1);
        const long long ta = mp.prof ? clock64() : 0;
        usep ^= 3u;
        tc_fence_after();
        const uint32_t tb = tmem_base_ld() + uint32_t(jh * 256) + (uint32_t(q * 32) << 16);
        const int nsteps = min(256, P.N - nb * 256) / 64;
        uint32_t pk[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < nsteps) {
            uint32_t r[64];
            if (DIAG(mp) & 2) {
#pragma unroll
              for (int i = 0; i < 64; ++i) r[i] = uint32_t(i * lane);
            } else {
              TMEM_LD32(tb + uint32_t(c * 64), r);
              TMEM_LD32(tb + uint32_t(c * 64 + 32), (r + 32));
              tmem_wait_ld();
            }
            if (DIAG(mp) & 1) {
#pragma unroll
              for (int i = 0; i < 32; ++i) pk[c * 32 + i] = __byte_perm(r[2 * i], r[2 * i + 1], 0x7632);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                __nv_bfloat162 v = __floats2bfloat162_rn(P.lam * __uint_as_float(r[2 * i]), P.lam * __uint_as_float(r[2 * i + 1]));
                pk[c * 32 + i] = *reinterpret_cast<uint32_t*>(&v);
              }
            }
          }
        }
        const long long tb2 = mp.prof ? clock64() : 0;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_n(tempty_leader0 + uint32_t(jh * 8), 2);
        if (mp.prof) { ep_a += tb2 - ta; ep_b += clock64() - tb2; ++ep_n; }
        const int row0 = mb * 512 + int(rank) * 256 + jh * BM + q * 32;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < nsteps) {
            if (P.act) {   // dX = bf16(dh) * act'(U): U's 32 x 64 chunk by TMA into this warp's buffer
              if (lane == 0) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                mbar_expect_tx(&ubar[warp - EPI_WARP0], 4096);
                tma_load_2d<1>(&maps.u, buf, smem_u32(&ubar[warp - EPI_WARP0]), nb * 256 + c * 64, row0);
              }
              mbar_wait(&ubar[warp - EPI_WARP0], uph);
              uph ^= 1;
#pragma unroll
              for (int cc = 0; cc < 8; ++cc) {
                uint32_t w0, w1, w2, w3;
                const uint32_t a = smem_u32(buf + lane * 128 + ((cc ^ (lane & 7)) << 4));
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(a));
                const uint32_t uw[4] = {w0, w1, w2, w3};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 d = unpack_bf2(pk[c * 32 + 4 * cc + e]), x = unpack_bf2(uw[e]);
                  pk[c * 32 + 4 * cc + e] = pack_bf2(d.x * gelu_tanh_grad(x.x), d.y * gelu_tanh_grad(x.y));
                }
              }
              __syncwarp();   // every row read before the buffer takes dX
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const uint32_t a = smem_u32(buf + lane * 128 + ((cc ^ (lane & 7)) << 4));
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pk[c * 32 + 4 * cc]),
                           "r"(pk[c * 32 + 4 * cc + 1]), "r"(pk[c * 32 + 4 * cc + 2]), "r"(pk[c * 32 + 4 * cc + 3])
                           : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                               reinterpret_cast<uint64_t>(&maps.b[prob])),
                           "r"(nb * 256 + c * 64), "r"(row0), "r"(smem_u32(buf))
                           : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          }
        }
        if (P.publish) {   // this warp's 32 rows of the tile are in global memory: release them
          if (lane == 0) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(mp.flags + u) : "memory");
          }
          __syncwarp();
        }
      } else {
        // DW: this warp's 32 rows (hash-tile row x) x 128 columns (hash tiles y = 4 nb + 2 jh, +1)
        const int h = dwh;
        dwh ^= 1;
        const int rb = mb * 256 + int(rank) * 128 + q * 32;
        int64_t t_off = 0;
        float t_scale = 0.f;
        {
          const int y = nb * 4 + (lane & 3);
          if (lane < 4 && rb < P.M && y * 64 < P.N) {
            const int t = (rb >> 6) * P.ny + y;
            // deterministic: the tile's slot in the workspace (reduced in fixed order afterwards)
            t_off = P.ws_slot >= 0 ? (int64_t(split) * P.ntiles + t) * 4096 : P.off[t];
            t_scale = P.sgn[t] < 0 ? -P.lam : P.lam;
          }
        }
        mbar_wait(&tfull[h], (usep >> h) & 1);
        usep ^= 1u << h;
        tc_fence_after();
        const uint32_t tb = tmem_base_ld() + uint32_t(h * 256) + (uint32_t(q * 32) << 16);
        const int nvalid = min(256, P.N - nb * 256) / 32;
#pragma unroll 1
        for (int c = jh * 4; c < jh * 4 + 4; ++c) {
          const float scale = __shfl_sync(0xffffffffu, t_scale, c >> 1);
          const int64_t tbo = __shfl_sync(0xffffffffu, t_off, c >> 1);
          if (c >= nvalid) continue;
          uint32_t r[32];
          TMEM_LD32(tb + uint32_t(c * 32), r);
          tmem_wait_ld();
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) {
            const uint32_t a = smem_u32(buf + lane * 128 + ((cc ^ (lane & 7)) << 4));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                         "r"(__float_as_uint(scale * __uint_as_float(r[4 * cc]))),
                         "r"(__float_as_uint(scale * __uint_as_float(r[4 * cc + 1]))),
                         "r"(__float_as_uint(scale * __uint_as_float(r[4 * cc + 2]))),
                         "r"(__float_as_uint(scale * __uint_as_float(r[4 * cc + 3])))
                         : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0 && rb < P.M) {   // 32 rows x 32 fp32 of one hash tile
            const int x0 = (c & 1) * 32;
            const int y0 = int(tbo >> 6) + (rb & 63) + (P.ws_slot >= 0 ? 0 : drow);
            if (P.ws_slot >= 0)   // deterministic: plain store into the per-tile workspace
              asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                               reinterpret_cast<uint64_t>(&maps.ws[P.ws_slot])),
                           "r"(x0), "r"(y0), "r"(smem_u32(buf))
                           : "memory");
            else                  // fast: TMA reduce-add into dM in L2
              asm volatile(
                  "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                      reinterpret_cast<uint64_t>(&maps.dm.m[(tbo >> 3) & 7])),
                  "r"(x0), "r"(y0), "r"(smem_u32(buf))
                  : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_n(tempty_leader0 + uint32_t(h * 8), 1);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }

  if (mp.prof && lane == 0) {   // [cta][8]: total, producer dep wait, MMA wait full / TMEM in DX, in DW units,
    long long* o = mp.prof + blockIdx.x * 8;   // DX TMEM->register phase (warp 4), DX units drained (warp 4)
    if (warp == 0) { o[0] = clock64() - t_start; }
    if (warp == 1 && leader) { o[2] = mw_full; o[3] = mw_tmem; o[4] = mw_full_dw; o[5] = mw_tmem_dw; }
    if (warp == EPI_WARP0) { o[6] = ep_a; o[7] = ep_n; o[1] = ep_b; }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_ld()), "r"(TMEM_COLS));
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // a driver-API call: the calling thread needs a current context, which a thread that has made
  // no runtime call yet lacks (torch's autograd worker running a backward that starts with a
  // tensor-map build: CUDA_ERROR_INVALID_CONTEXT).  cudaSetDevice makes the primary one current.
  thread_local bool ctx_ready = false;
  if (!ctx_ready) {
    int d = 0;
    if (cudaGetDevice(&d) == cudaSuccess) cudaSetDevice(d);
    ctx_ready = true;
  }
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 2-D tensor [rows x cols] (cols contiguous, bf16 or fp32), box {box_c, box_r}, SWIZZLE_128B.
roast_status_t make_map_2d(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t row_bytes,
                           uint32_t box_c, uint32_t box_r, bool fp32 = false) {
  auto fn = encode_fn();
  if (!fn) return fail(ROAST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_c, box_r};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ROAST_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return ROAST_OK;
}

// 3-D view of a row-major bf16 [rows x cols] tensor as {64 cols, rows, cols / 64 blocks}: one box
// {64, box_r, nblk} fetches nblk 64-wide column blocks, each landing as its own [box_r x 128 B]
// SW128 atom column — the MN-major operand layout — in a single TMA operation.
roast_status_t make_map_blocks(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_r,
                               uint32_t nblk) {
  auto fn = encode_fn();
  if (!fn) return fail(ROAST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, rows, cols / 64};
  cuuint64_t strides[2] = {cols * 2, 128};
  cuuint32_t box[3] = {64, box_r, nblk};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ROAST_ERR_CUDA, "cuTensorMapEncodeTiled(3d) failed (" + std::to_string(int(r)) + ")");
  return ROAST_OK;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int cta_group() {
  static int cg = 0;
  if (!cg) {
    const char* e = getenv("ROAST_CTA_GROUP");
    cg = (e && atoi(e) == 1) ? 1 : 2;
  }
  return cg;
}

template <int MODE, int CG, int WM, bool CHAIN = false, int NU = BN, bool ACT = false, bool XBUF = false>
roast_status_t launch_cg(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& o, const WMaps& w,
                         const Params& p, const CUtensorMap& a1, const CUtensorMap& o1, const Params& p1,
                         int grid_pairs, cudaStream_t s, const WMapsHalf* hw = nullptr,
                         const CUtensorMap* act_map = nullptr) {
  using C = Cfg<CG, WM, NU, XBUF>;
  static std::atomic<unsigned long long> attr{0};   // smem opt-in, once per device
  if (first_on_device(attr)) {
    cudaError_t e =
        cudaFuncSetAttribute(roast_mm_sm100<MODE, CG, WM, CHAIN, NU, ACT, XBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(smem)");
  }
  const int pairs = grid_pairs > 0 ? grid_pairs : std::min(p.units, num_sms() / CG);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(pairs * CG));
  cfg.blockDim = dim3(Roles<MODE, CG, WM>::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see griddepcontrol in the kernel
  at[1].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = !(getenv("ROAST_PDL") && atoi(getenv("ROAST_PDL")) == 0);
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  static long long* prof = nullptr;
  Params pp = p, pp1 = p1;
  if (const char* e = getenv("ROAST_EPI")) pp.epi = atoi(e);
  if (const char* e = getenv("ROAST_EXP")) pp.exp = pp1.exp = atoi(e);
  if (getenv("ROAST_PROF")) {
    if (!prof) cudaMallocManaged(&prof, sizeof(long long) * 8 * 512);
    cudaMemset(prof, 0, sizeof(long long) * 8 * 512);
    pp.prof = prof;
    pp1.prof = prof;
  }
  static const WMapsHalf no_half{};
  cudaError_t e = cudaLaunchKernelEx(&cfg, roast_mm_sm100<MODE, CG, WM, CHAIN, NU, ACT, XBUF>, a, b, o, w, pp, a1, o1, pp1,
                                     hw ? *hw : no_half, act_map ? *act_map : o);
  if (e != cudaSuccess) return cuda_fail(e, "roast_mm_sm100 launch");
  if (pp.prof) {
    cudaDeviceSynchronize();
    double acc[8] = {0};
    long long mx = 0;
    for (int i = 0; i < pairs * CG; ++i) {
      for (int k = 0; k < 8; ++k) acc[k] += double(prof[i * 8 + k]);
      mx = std::max(mx, prof[i * 8 + 5]);
    }
    const int n = pairs * CG, nl = (pairs * CG + CG - 1) / CG;
    if (Roles<MODE, CG, WM>::RF)   // register-held epilogue: slot 0 = MMA wait for TMEM, 6 = TMEM->RF phase
      fprintf(stderr, "[roast prof] RF wm %d mode %d nu %d units %d kb %d | total %.0f (max %lld) | mma wait-tmem %.0f "
              "mma wait-full %.0f | %.0f MHz | epi busy %.0f (tmem->rf %.0f)  (cycles, mean/CTA)\n",
              WM, MODE, NU, p.units, p.k_blocks, acc[5] / n, mx, acc[0] / nl, acc[1] / nl,
              acc[5] / (acc[3] > 0 ? acc[3] : 1) * 1e3, acc[4] / n, acc[6] / n);
    else
    fprintf(stderr, "[roast prof] dw3d %d wm %d mode %d cg %d units %d kb %d | total %.0f (max %lld) | epi-fence %.0f | "
            "mma wait-full %.0f epi-sts %.0f | %.0f MHz | epi busy %.0f (tmem %.0f, stg-wait %.0f)  (cycles, mean/CTA)\n",
            p.dw3d, WM, MODE, CG, p.units, p.k_blocks, acc[5] / n, mx, acc[0] / n, acc[1] / nl, acc[2] / nl, acc[5] / (acc[3] > 0 ? acc[3] : 1) * 1e3,
            acc[4] / n, acc[6] / n, acc[7] / n);
  }
  return ROAST_OK;
}

template <int MODE>
roast_status_t launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& o, const WMaps& w, Params p,
                      int wm, cudaStream_t s, int nu = BN, const WMapsHalf* hw = nullptr,
                      const CUtensorMap* o_act = nullptr) {
  if constexpr (MODE != DW) {
    if (p.act) {   // fused activation: the WM = 2 register-held epilogue (checked by the caller)
      // the activation's second tensor (mapAct): FWD writes act(Y) there, DX reads U from it.
      // The GELU dX epilogue is ALU-bound: it takes the second staging buffer (XBUF) so U chunk c + 1
      // loads while chunk c is computed (tools/act_probe.py, T = 65 536: 335 -> 302 us); the others
      // keep the fourth pipeline stage (residual dX 245 vs 237 us, forward 292 vs 283 us with XBUF)
      if constexpr (MODE == DX) {
        if (p.act == 1) {
          if (nu == 192) return launch_cg<MODE, 2, 2, false, 192, true, true>(a, b, o, w, p, a, o, p, 0, s, hw, o_act);
          return launch_cg<MODE, 2, 2, false, BN, true, true>(a, b, o, w, p, a, o, p, 0, s, nullptr, o_act);
        }
      }
      if (nu == 192) return launch_cg<MODE, 2, 2, false, 192, true>(a, b, o, w, p, a, o, p, 0, s, hw, o_act);
      return launch_cg<MODE, 2, 2, false, BN, true>(a, b, o, w, p, a, o, p, 0, s, nullptr, o_act);
    }
    if (nu == 192) return launch_cg<MODE, 2, 2, false, 192>(a, b, o, w, p, a, o, p, 0, s, hw);
  }
  if (cta_group() == 1) return launch_cg<MODE, 1, 1>(a, b, o, w, p, a, o, p, 0, s);
  return wm == 2 ? launch_cg<MODE, 2, 2>(a, b, o, w, p, a, o, p, 0, s)
                 : launch_cg<MODE, 2, 1>(a, b, o, w, p, a, o, p, 0, s);
}

}  // namespace sm100

using namespace sm100;


roast_status_t sm100_prepare(Ctx* c) {
  if (c->tmap_shadow_valid) return ROAST_OK;
  static_assert(sizeof(WMaps) <= sizeof(Ctx::tmap_shadow), "tmap storage");
  static_assert(sizeof(WMapsHalf) <= sizeof(Ctx::tmap_shadow_half), "tmap storage");
  WMaps* w = reinterpret_cast<WMaps*>(c->tmap_shadow);
  WMapsHalf* hw = reinterpret_cast<WMapsHalf*>(c->tmap_shadow_half);
  for (int r = 0; r < 8; ++r) {
    const int64_t elems = c->shadow_reps * c->shadow_elems - 8 * r;   // every replica
    roast_status_t st = make_map_2d(&w->m[r], c->shadow + 8 * r, 64, uint64_t(elems / 64), 128, 64, 64);
    if (st) return st;
    st = make_map_2d(&hw->m[r], c->shadow + 8 * r, 64, uint64_t(elems / 64), 128, 64, 32);
    if (st) return st;
  }
  c->tmap_shadow_valid = true;
  return ROAST_OK;
}

static bool supported(const Ctx* c, const Module& m) {
  return m.d_coord_xy != nullptr && c->cfg.tile_layout == ROAST_ROW_MAJOR && c->tile.z1 == 64 &&
         c->tile.z2 == 64 && m.H % 64 == 0 && m.O % 64 == 0;
}

static Params base_params(const Ctx* c, const Module& m, int64_t T) {
  Params p{};
  p.T = T;
  p.off = m.d_off;
  p.sgn = m.d_sgn;
  p.ny = m.ny;
  p.neg_row = c->neg_base / 64;
  p.reps = c->shadow_reps;
  p.rep_rows = int(c->shadow_elems / 64);
  p.lam = m.lam;
  p.ntiles = m.nx * m.ny;
  p.splits = 1;
  return p;
}

// WM (M sub-tiles per CTA) from a makespan model: WM = 2 halves the TMA box rate per
// MMA (one 256-row A box + the same B feeds two MMAs) but doubles the unit size and
// exposes the epilogue (single-buffered accumulator).  eff = measured MMA-busy share.
static int choose_wm(int64_t m_rows, int n_tiles, int splits) {
  if (const char* e = getenv("ROAST_WM")) return atoi(e) == 2 ? 2 : 1;
  if (cta_group() != 2) return 1;
  const int pairs = num_sms() / 2;
  auto cost = [&](int wm, double eff) {
    const int64_t units = ((m_rows + 256 * wm - 1) / (256 * wm)) * n_tiles * splits;
    return double((units + pairs - 1) / pairs) * wm / eff;
  };
  return cost(2, 0.85) < cost(1, 0.6) ? 2 : 1;
}

// ---- autotuner (NEXT #4) ---------------------------------------------
// The paper autotunes its Triton tile per layer shape with two strategies: inference-
// optimal (tune the forward, share its tile with the backward kernels) and training-
// optimal (tune forward and backward kernels together).  Here the hash tile is part of
// the model (64 x 64, R10), so what is tuned is the kernel configuration: WM (M sub-tiles
// per CTA pair) for FWD / DX and (WM, split-K) for DW.  Each candidate is timed once with
// CUDA events on the caller's stream (1 warm-up + 3 timed launches) the first time a
// shape is seen outside stream capture; the winner is cached per (kernel, H, O, tokens).
namespace {
enum { kTuneFwd = 0, kTuneDx = 1, kTuneDw = 2 };

std::array<int64_t, 4> tune_key(int kind, const Module& m, int64_t T) { return {kind, m.H, m.O, T}; }

bool can_tune(const Ctx* c, cudaStream_t s) {
  if (c->autotune == ROAST_TUNE_OFF) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
}

template <class F>
float time_candidate(F&& f, cudaStream_t s) {
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess) return -1.f;
  if (cudaEventCreate(&e1) != cudaSuccess) {
    cudaEventDestroy(e0);
    return -1.f;
  }
  float ms = -1.f;
  if (f() == ROAST_OK) {   // warm-up (also sets smem attributes / builds descriptors)
    bool ok = cudaEventRecord(e0, s) == cudaSuccess;
    for (int r = 0; r < 3 && ok; ++r) ok = f() == ROAST_OK;
    ok = ok && cudaEventRecord(e1, s) == cudaSuccess && cudaEventSynchronize(e1) == cudaSuccess;
    if (ok && cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) ms = -1.f;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}
}  // namespace

// FWD / DX share the geometry: M = tokens, N = the module's output side, K = its input side.
// nu = output columns per unit (256, or 192 for DX with WM = 2).
static roast_status_t tok_major_launch(Ctx* c, const Module& m, const void* A, void* out, int64_t T, int N, int K,
                                       const int32_t* coord, int coord_ld, bool dx, int wm, const float* bias,
                                       cudaStream_t s, int nu = BN, int act = 0, const void* act_in = nullptr,
                                       void* act_out = nullptr) {
  if (act && (wm != 2 || cta_group() != 2)) return ROAST_ERR_UNSUPPORTED;   // the RF epilogue only
  CUtensorMap a;
  roast_status_t st = make_map_2d(&a, A, uint64_t(K), uint64_t(T), uint64_t(K) * 2, BK, BM * wm);
  if (st) return st;
  Params p = base_params(c, m, T);
  p.M = int(std::min<int64_t>(T, 1 << 30));
  p.N = N;
  p.K = K;
  p.m_tiles = int((T + BM * cta_group() * wm - 1) / (BM * cta_group() * wm));
  p.n_tiles = (p.N + nu - 1) / nu;
  p.k_blocks = p.K / BK;
  p.kb_per_split = p.k_blocks;
  p.units = p.m_tiles * p.n_tiles;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.bias = dx ? nullptr : bias;
  p.coord = coord;
  p.coord_ld = coord_ld;
  p.act = act;
  p.act_in = static_cast<const __nv_bfloat16*>(act_in);
  p.act_out = static_cast<__nv_bfloat16*>(act_out);
  CUtensorMap o;   // output [T x N] bf16, stored 32 rows x 64 columns per TMA op
  st = make_map_2d(&o, out, uint64_t(N), uint64_t(T), uint64_t(N) * 2, 64, 32);
  if (st) return st;
  const WMaps& w = *reinterpret_cast<const WMaps*>(c->tmap_shadow);
  const WMapsHalf* hw = reinterpret_cast<const WMapsHalf*>(c->tmap_shadow_half);
  CUtensorMap o2 = o;   // with an activation (the kernel's mapAct): FWD its output, DX the U input, 32 x 64 boxes
  if (act && (st = make_map_2d(&o2, dx ? act_in : act_out, uint64_t(N), uint64_t(T), uint64_t(N) * 2, 64, 32)))
    return st;
  st = dx ? launch<DX>(a, a, o, w, p, wm, s, nu, hw, &o2) : launch<FWD>(a, a, o, w, p, wm, s, nu, hw, &o2);
  if (!st) c->launches++;
  return st;
}

// (WM, N per unit) configurations a FWD / DX launch may use; the tuned map stores N / 64 in
// the `splits` slot (legacy 1 = 256)
static bool nu192_ok(bool dx, int wm, int N) { (void)dx; return wm == 2 && cta_group() == 2 && N % 192 == 0; }

// makespan model (no tuning): rounds of units over the CTA pairs x per-unit MMA work
static void choose_tok_major(int64_t T, int N, bool dx, int& wm, int& nu) {
  wm = choose_wm(T, (N + BN - 1) / BN, 1);
  nu = BN;
  if (nu192_ok(dx, wm, N) && !getenv("ROAST_NO_NU192")) {
    const int pairs = num_sms() / 2;
    const int64_t mt = (T + 511) / 512;
    const double c256 = double((mt * ((N + 255) / 256) + pairs - 1) / pairs) * 256;
    const double c192 = double((mt * (N / 192) + pairs - 1) / pairs) * 192;
    if (c192 < c256) nu = 192;
  }
}

static roast_status_t run_tok_major(Ctx* c, const Module& m, const void* A, void* out, int64_t T, int N, int K,
                                    const int32_t* coord, int coord_ld, bool dx, const float* bias, cudaStream_t s,
                                    int act = 0, const void* act_in = nullptr, void* act_out = nullptr) {
  if (!supported(c, m) || T >= (int64_t(1) << 31)) return ROAST_ERR_UNSUPPORTED;
  if (act) {   // the fused activation lives in the WM = 2 register-held epilogue: WM = 2, N per unit tuned
    if (cta_group() != 2) return ROAST_ERR_UNSUPPORTED;
    roast_status_t st = sm100_prepare(c);
    if (st) return st;
    const auto key = tune_key((dx ? kTuneDx : kTuneFwd) + 16, m, T);   // its own cache entry
    auto it = c->tuned.find(key);
    int nu = BN;
    if (it != c->tuned.end()) {
      nu = it->second.second == 3 ? 192 : BN;
    } else if (nu192_ok(dx, 2, N) && can_tune(c, s)) {
      const float t256 = time_candidate([&] {
        return tok_major_launch(c, m, A, out, T, N, K, coord, coord_ld, dx, 2, bias, s, BN, act, act_in, act_out); }, s);
      const float t192 = time_candidate([&] {
        return tok_major_launch(c, m, A, out, T, N, K, coord, coord_ld, dx, 2, bias, s, 192, act, act_in, act_out); }, s);
      nu = (t192 >= 0.f && t192 < t256) ? 192 : BN;
      c->tuned[key] = {2, nu / 64};
    }
    return tok_major_launch(c, m, A, out, T, N, K, coord, coord_ld, dx, 2, bias, s, nu, act, act_in, act_out);
  }
  roast_status_t st = sm100_prepare(c);
  if (st) return st;
  const auto key = tune_key(dx ? kTuneDx : kTuneFwd, m, T);
  auto it = c->tuned.find(key);
  auto fwd = c->tuned.find(tune_key(kTuneFwd, m, T));
  int wm, nu;
  choose_tok_major(T, N, dx, wm, nu);
  if (it != c->tuned.end()) {
    wm = it->second.first;
    nu = it->second.second == 3 && nu192_ok(dx, wm, N) ? 192 : BN;
  } else if (dx && c->autotune == ROAST_TUNE_INFERENCE && fwd != c->tuned.end()) {
    wm = fwd->second.first;   // inference-optimal: the backward shares the forward's tile
    nu = BN;
  } else if ((!dx || c->autotune == ROAST_TUNE_TRAINING) && can_tune(c, s)) {
    float best = 1e30f;
    for (int w = 1; w <= (cta_group() == 2 ? 2 : 1); ++w)
      for (int u : {BN, 192}) {
        if (u == 192 && !nu192_ok(dx, w, N)) continue;
        const float ms = time_candidate(
            [&] { return tok_major_launch(c, m, A, out, T, N, K, coord, coord_ld, dx, w, bias, s, u); }, s);
        if (ms >= 0.f && ms < best) {
          best = ms;
          wm = w;
          nu = u;
        }
      }
    c->tuned[key] = {wm, nu / 64};
  }
  return tok_major_launch(c, m, A, out, T, N, K, coord, coord_ld, dx, wm, bias, s, nu);
}

roast_status_t sm100_fwd(Ctx* c, const Module& m, const void* X, void* Y, int64_t T, const float* bias,
                         cudaStream_t s) {
  return run_tok_major(c, m, X, Y, T, int(m.O), int(m.H), m.d_coord_xy, m.ny, false, bias, s);
}

roast_status_t sm100_dx(Ctx* c, const Module& m, const void* dY, void* dX, int64_t T, cudaStream_t s) {
  return run_tok_major(c, m, dY, dX, T, int(m.H), int(m.O), m.d_coord_yx, m.nx, true, nullptr, s);
}

roast_status_t sm100_fwd_act(Ctx* c, const Module& m, const void* X, void* Y, void* A, int64_t T, const float* bias,
                             int act, cudaStream_t s) {
  return run_tok_major(c, m, X, Y, T, int(m.O), int(m.H), m.d_coord_xy, m.ny, false, bias, s, act, nullptr, A);
}

roast_status_t sm100_dx_act(Ctx* c, const Module& m, const void* dY, const void* U, void* dX, int64_t T, int act,
                            cudaStream_t s) {
  return run_tok_major(c, m, dY, dX, T, int(m.H), int(m.O), m.d_coord_yx, m.nx, true, nullptr, s, act, U, nullptr);
}

// ---- chained pair of GEMMs ------------------------------------------------------
// Problem 0 (N0 = 4 * 64 * n_tiles0 output columns) feeds problem 1 as its A operand
// (K1 = N0).  Alone, each launch is quantised on its own: C2's 3072 -> 768 GEMM has 48
// units for 74 CTA pairs and the 768 -> 3072 one 192 units (2.6 rounds).  Chained, the
// second GEMM's units start on the pairs the first leaves idle and stream their K loop
// behind the first GEMM's output tiles (per-tile ready counters).  The static per-pair
// schedule comes from a list-scheduling simulation in k-block time units (an MMA k-block
// of a WM = 2 unit ~ 1024 clk; per-unit epilogue exposure EPI); every pair runs all its
// problem-0 units before any problem-1 unit, which keeps the waits deadlock-free.
namespace {
struct ChainPlan {
  std::vector<int32_t> sched;   // [pairs][len], -1 padded
  int len = 0;
  double makespan = 0, sequential = 0;
};

ChainPlan plan_chain(int m_tiles, int nt0, int kb0, int nt1, int kb1, int npairs) {
  double EPI = 5.0, LAT = 1.0;
  if (const char* e = getenv("ROAST_CHAIN_EPI")) EPI = atof(e);   // planner-model experiments
  if (const char* e = getenv("ROAST_CHAIN_LAT")) LAT = atof(e);
  const int units0 = m_tiles * nt0, units1 = m_tiles * nt1;
  const double c0 = kb0 + EPI, c1 = kb1 + EPI;
  ChainPlan best;
  best.makespan = 1e30;
  best.sequential = double((units0 + npairs - 1) / npairs) * c0 + double((units1 + npairs - 1) / npairs) * c1;
  const int n2 = std::min(npairs, units1);   // pairs that run problem-1 units
  // problem-0 units in m-major or n-major order (n-major completes the K groups every
  // problem-1 unit needs first, so all of them can stream early); k2 = problem-0 units on
  // each problem-1 pair before its problem-1 work
  for (int order = 0; order < 2; ++order)
    for (int k2 = 0; k2 <= 8; ++k2) {
      std::vector<double> free_t(npairs, 0.0), fin0(units0, 0.0);
      std::vector<int> cnt0(npairs, 0);
      std::vector<std::vector<int32_t>> lists(npairs);
      for (int i = 0; i < units0; ++i) {
        const int u = order == 0 ? i : (i % m_tiles) * nt0 + i / m_tiles;
        int pick = -1;
        for (int q = 0; q < npairs; ++q) {
          if (q < n2 && cnt0[q] >= k2 && n2 < npairs) continue;
          if (pick < 0 || free_t[q] < free_t[pick]) pick = q;
        }
        fin0[u] = free_t[pick] + c0;
        free_t[pick] = fin0[u];
        cnt0[pick]++;
        lists[pick].push_back(u);
      }
      for (int u = 0; u < units1; ++u) {
        const int mb = u / nt1;
        int pick = 0;
        for (int q = 1; q < n2; ++q)
          if (free_t[q] < free_t[pick]) pick = q;
        double t = free_t[pick];
        for (int g = 0; g < nt0; ++g) t = std::max(t, fin0[mb * nt0 + g] + LAT) + double(kb1) / nt0;
        free_t[pick] = t + EPI;
        lists[pick].push_back((1 << 24) | u);
      }
      const double mk = *std::max_element(free_t.begin(), free_t.end());
      if (mk < best.makespan - 1e-9) {
        best.makespan = mk;
        best.len = 0;
        for (auto& l : lists) best.len = std::max<int>(best.len, int(l.size()));
        best.sched.assign(size_t(npairs) * best.len, -1);
        for (int q = 0; q < npairs; ++q)
          for (size_t i = 0; i < lists[q].size(); ++i) best.sched[size_t(q) * best.len + i] = lists[q][i];
      }
    }
  return best;
}
}  // namespace

roast_status_t sm100_chain(Ctx* c, const Module& m0, const Module& m1, const void* A0, void* out0, void* out1,
                           int64_t T, bool dx, const float* bias0, const float* bias1, cudaStream_t s, int act,
                           void* act_buf) {
  if (!supported(c, m0) || !supported(c, m1) || cta_group() != 2 || T >= (int64_t(1) << 31) || T <= 0)
    return ROAST_ERR_UNSUPPORTED;
  if (act && dx) return ROAST_ERR_UNSUPPORTED;   // forward only: problem 1 reads act(problem 0's output)
  if (getenv("ROAST_NO_CHAIN")) return ROAST_ERR_UNSUPPORTED;
  // geometry: FWD problem 0 = m0 (K = H0, N = O0), problem 1 = m1 (K = H1 = O0, N = O1);
  //           DX  problem 0 = m0 (K = O0, N = H0), problem 1 = m1 (K = O1 = H0, N = H1)
  const int N0 = int(dx ? m0.H : m0.O), K0 = int(dx ? m0.O : m0.H);
  const int N1 = int(dx ? m1.H : m1.O), K1 = int(dx ? m1.O : m1.H);
  if (K1 != N0 || N0 % BN) return ROAST_ERR_UNSUPPORTED;   // problem-0 tiles must cover whole 4-k-block groups
  constexpr int WMC = 2;
  const int pairs = num_sms() / 2;
  const int m_tiles = int((T + BM * 2 * WMC - 1) / (BM * 2 * WMC));
  const int nt0 = N0 / BN, nt1 = (N1 + BN - 1) / BN;
  const std::array<int64_t, 6> key{dx ? 1 : 0, m0.H, m0.O, m1.H, m1.O, T};
  auto it = c->chain_plans.find(key);
  if (it == c->chain_plans.end()) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return ROAST_ERR_UNSUPPORTED;   // planning allocates; plan on an eager call first
    ChainPlan plan = plan_chain(m_tiles, nt0, K0 / BK, nt1, K1 / BK, pairs);
    int32_t* d = nullptr;
    // the waits assume every CTA pair of the grid is resident at once: chain only if the
    // device can hold all `pairs` clusters of this kernel together
    bool resident = false;
    {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(unsigned(2 * pairs));
      q.blockDim = dim3(Roles<FWD, 2, WMC>::THREADS);
      q.dynamicSmemBytes = Cfg<2, WMC>::SMEM;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 2;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      q.attrs = a;
      q.numAttrs = 1;
      auto kfn = dx ? roast_mm_sm100<DX, 2, WMC, true> : roast_mm_sm100<FWD, 2, WMC, true>;
      int nclusters = 0;
      if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<2, WMC>::SMEM) == cudaSuccess &&
          cudaOccupancyMaxActiveClusters(&nclusters, kfn, &q) == cudaSuccess)
        resident = nclusters >= pairs;
      cudaGetLastError();
      if (getenv("ROAST_VERBOSE"))
        fprintf(stderr, "[roast] chain %s: max co-resident clusters %d, grid %d pairs\n", dx ? "dx" : "fwd", nclusters,
                pairs);
    }
    if (resident && plan.makespan < 0.97 * plan.sequential) {
      ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&d), plan.sched.size() * sizeof(int32_t)));
      ROAST_CUDA_CHECK(cudaMemcpy(d, plan.sched.data(), plan.sched.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    it = c->chain_plans.emplace(key, std::make_pair(d, plan.len)).first;
  }
  if (!it->second.first) return ROAST_ERR_UNSUPPORTED;
  // the ready counters of problem 0's tiles: the next of kChainSlots slots (chained launches
  // in flight on different streams never share counters); the slot array grows eagerly only
  const int64_t need = int64_t(m_tiles) * nt0;
  if (c->chain_slot_n < need) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return ROAST_ERR_UNSUPPORTED;   // first chained call of this size: make it eagerly
    ROAST_CUDA_CHECK(cudaDeviceSynchronize());   // the old slots may be in use
    cudaFree(c->chain_flags);
    c->chain_flags = nullptr;
    c->chain_slot_n = 0;
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->chain_flags), size_t(kChainSlots) * need * sizeof(int)));
    c->chain_slot_n = need;
  }
  int* flags = c->chain_flags + int64_t(c->chain_next++ % kChainSlots) * c->chain_slot_n;
  roast_status_t st = sm100_prepare(c);
  if (st) return st;
  auto prob = [&](const Module& m, const void* A, void* out, int N, int K, bool is_dx, const float* bias, Params& p,
                  CUtensorMap& ma, CUtensorMap& mo) -> roast_status_t {
    roast_status_t r = make_map_2d(&ma, A, uint64_t(K), uint64_t(T), uint64_t(K) * 2, BK, BM * WMC);
    if (r) return r;
    r = make_map_2d(&mo, out, uint64_t(N), uint64_t(T), uint64_t(N) * 2, 64, 32);
    if (r) return r;
    p = base_params(c, m, T);
    p.M = int(T);
    p.N = N;
    p.K = K;
    p.m_tiles = m_tiles;
    p.n_tiles = (N + BN - 1) / BN;
    p.k_blocks = K / BK;
    p.kb_per_split = p.k_blocks;
    p.units = p.m_tiles * p.n_tiles;
    p.out = reinterpret_cast<__nv_bfloat16*>(out);
    p.bias = is_dx ? nullptr : bias;
    p.coord = is_dx ? m.d_coord_yx : m.d_coord_xy;
    p.coord_ld = is_dx ? m.nx : m.ny;
    return ROAST_OK;
  };
  Params p0, p1;
  CUtensorMap a0, o0, a1, o1;
  if ((st = prob(m0, A0, out0, N0, K0, dx, bias0, p0, a0, o0))) return st;
  if ((st = prob(m1, act ? act_buf : out0, out1, N1, K1, dx, bias1, p1, a1, o1))) return st;
  CUtensorMap oact = o0;   // with an activation: problem 0 also writes act(Y_0) here, problem 1 reads it
  if (act) {
    if ((st = make_map_2d(&oact, act_buf, uint64_t(N0), uint64_t(T), uint64_t(N0) * 2, 64, 32))) return st;
    p0.act = act;
  }
  p0.chain = 1;
  p0.sched = it->second.first;
  p0.sched_len = it->second.second;
  p0.flags = flags;
  p0.err = c->d_err;
  ROAST_CUDA_CHECK(cudaMemsetAsync(flags, 0, size_t(p0.units) * sizeof(int), s));
  const WMaps& w = *reinterpret_cast<const WMaps*>(c->tmap_shadow);
  st = dx    ? launch_cg<DX, 2, WMC, true>(a0, a0, o0, w, p0, a1, o1, p1, pairs, s)
       : act ? launch_cg<FWD, 2, WMC, true, BN, true>(a0, a0, o0, w, p0, a1, o1, p1, pairs, s, nullptr, &oact)
             : launch_cg<FWD, 2, WMC, true>(a0, a0, o0, w, p0, a1, o1, p1, pairs, s);
  if (!st) c->launches++;
  return st;
}

// makespan model for DW: cost of (WM, split-K over tokens) = ceil(units / slots) * WM / (eff * s);
// eff = TMA-box-rate bound MMA share (4 boxes / 512 clk for WM 1, 6 / 1024 for WM 2)
static double dw_cost(const Module& m, int64_t T, int w, int sp) {
  const int cg = cta_group();
  const int slots = num_sms() / cg;
  const int n_tiles = int((m.O + BN - 1) / BN);
  const int tiles_w = int((m.H + BM * cg * w - 1) / (BM * cg * w)) * n_tiles;
  const double eff = w == 2 ? 0.95 : 0.9;   // measured MMA-busy share with 3-D operand boxes
  return double((int64_t(tiles_w) * sp + slots - 1) / slots) * w / (eff * sp);
}

// the split-K count with the lowest model cost (ties within 1e-9: the smaller count);
// skip = 1 gives the runner-up
static int dw_best_splits(const Module& m, int64_t T, int w, int skip = 0) {
  const int kb = int((T + BK - 1) / BK);
  int first = 0;
  for (int pass = 0; pass <= skip; ++pass) {
    int pick = 0;
    double best = 1e30;
    for (int sp = 1; sp <= std::min(kb, 16); ++sp) {
      if (pass == 1 && sp == first) continue;
      const double cst = dw_cost(m, T, w, sp);
      if (cst < best - 1e-9) {
        best = cst;
        pick = sp;
      }
    }
    if (pass == 0) first = pick;
    if (pass == skip) return pick ? pick : first;
  }
  return first;
}

static roast_status_t dw_launch(Ctx* c, const Module& m, const void* X, const void* dY, int64_t T, int wm, int splits,
                                cudaStream_t s) {
  CUtensorMap a, b;
  roast_status_t st = make_map_2d(&a, X, uint64_t(m.H), uint64_t(T), uint64_t(m.H) * 2, 64, BK);
  if (st) return st;
  st = make_map_2d(&b, dY, uint64_t(m.O), uint64_t(T), uint64_t(m.O) * 2, 64, BK);
  if (st) return st;
  const int cg = cta_group();
  Params p = base_params(c, m, T);
  p.M = int(m.H);
  p.N = int(m.O);
  p.n_tiles = (p.N + BN - 1) / BN;
  p.k_blocks = int((T + BK - 1) / BK);
  p.m_tiles = (p.M + BM * cg * wm - 1) / (BM * cg * wm);
  const int tiles = p.m_tiles * p.n_tiles;
  // one 3-D box per operand per stage (falls back to 64x64 2-D boxes if the driver rejects the view)
  if (!getenv("ROAST_DW2D")) {
    CUtensorMap a3, b3;
    if (make_map_blocks(&a3, X, uint64_t(m.H), uint64_t(T), BK, 2 * wm) == ROAST_OK &&
        make_map_blocks(&b3, dY, uint64_t(m.O), uint64_t(T), BK, 4 / cg) == ROAST_OK) {
      a = a3;
      b = b3;
      p.dw3d = 1;
    }
  }
  p.kb_per_split = (p.k_blocks + splits - 1) / splits;
  splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;   // no empty splits
  p.splits = splits;
  p.units = tiles * splits;
  p.dM = c->dM;
  const bool det = c->cfg.deterministic != 0;
  Scratch ws;   // deterministic: per-tile partials, freed (stream-ordered) after the reduce
  if (det) {
    st = scratch_alloc(ws, size_t(splits) * p.ntiles * 4096 * sizeof(float), s);
    if (st) return st;
    p.ws = ws.as<float>();
  }
  // dM viewed as 8 [rows x 64] fp32 tensors, one per 32-byte phase (tile offsets are multiples of A = 8)
  CUtensorMap o;
  WMaps& dmaps = *reinterpret_cast<WMaps*>(c->tmap_dm);
  memset(&o, 0, sizeof(o));
  if (det) {
    const uint64_t rows = uint64_t(splits) * p.ntiles * 64;
    st = make_map_2d(&o, p.ws, 64, rows, 256, 32, 32, true);
    if (st) return st;
  } else if (c->tmap_dm_for != c->dM) {   // cached until dM is rebound
    for (int r = 0; r < 8; ++r) {
      const int64_t elems = c->mem_size - 8 * r;
      st = make_map_2d(&dmaps.m[r], c->dM + 8 * r, 64, uint64_t(elems / 64), 256, 32, 32, true);
      if (st) return st;
    }
    c->tmap_dm_for = c->dM;
  }
  st = launch<DW>(a, b, o, dmaps, p, wm, s);
  if (st) return st;
  c->launches++;
  if (det) {
    cudaError_t e = launch_det_reduce(c, m, p.ws, splits, s);
    if (e != cudaSuccess) return cuda_fail(e, "det_reduce");
    c->launches++;
  }
  return ROAST_OK;
}

roast_status_t sm100_dw(Ctx* c, const Module& m, const void* X, const void* dY, int64_t T, cudaStream_t s) {
  if (!supported(c, m) || T >= (int64_t(1) << 31)) return ROAST_ERR_UNSUPPORTED;
  const int wmax = cta_group() == 2 ? 2 : 1;
  int wm = 1, splits = 1;
  const auto key = tune_key(kTuneDw, m, T);
  auto it = c->tuned.find(key);
  auto fwd = c->tuned.find(tune_key(kTuneFwd, m, T));
  const char* ewm = getenv("ROAST_WM");
  {   // the makespan model's choice (also the fallback of the tuner)
    double best = 1e30;
    for (int w = 1; w <= wmax; ++w) {
      if (ewm && atoi(ewm) != w) continue;
      const int sp = dw_best_splits(m, T, w);
      if (dw_cost(m, T, w, sp) < best - 1e-9) {
        best = dw_cost(m, T, w, sp);
        wm = w;
        splits = sp;
      }
    }
  }
  if (it != c->tuned.end()) {
    wm = it->second.first;
    splits = it->second.second;
  } else if (c->autotune == ROAST_TUNE_INFERENCE && fwd != c->tuned.end() && fwd->second.first <= wmax) {
    wm = fwd->second.first;   // inference-optimal: share the forward's tile, model picks split-K
    splits = dw_best_splits(m, T, wm);
  } else if (c->autotune == ROAST_TUNE_TRAINING && can_tune(c, s)) {
    // every timed candidate accumulates into dM: snapshot it and restore afterwards
    float* save = nullptr;
    ROAST_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&save), c->mem_size * sizeof(float), s));
    ROAST_CUDA_CHECK(cudaMemcpyAsync(save, c->dM, c->mem_size * sizeof(float), cudaMemcpyDeviceToDevice, s));
    float best = 1e30f;
    const int kbt = int((T + BK - 1) / BK);
    for (int w = 1; w <= wmax; ++w)
      for (int sp : {1, 2, 3, 4, 6, 8, 12, 16}) {   // the model ignores epilogue exposure: time them all
        if (sp > kbt) continue;
        const float ms = time_candidate([&] { return dw_launch(c, m, X, dY, T, w, sp, s); }, s);
        if (ms >= 0.f && ms < best) {
          best = ms;
          wm = w;
          splits = sp;
        }
      }
    cudaError_t e = cudaMemcpyAsync(c->dM, save, c->mem_size * sizeof(float), cudaMemcpyDeviceToDevice, s);
    cudaFreeAsync(save, s);
    if (e != cudaSuccess) return cuda_fail(e, "autotune dM restore");
    c->tuned[key] = {wm, splits};
  }
  return dw_launch(c, m, X, dY, T, wm, splits, s);
}

}  // namespace roast

// ---- fused backward of a chained pair (roast_linear_bwd_chain) ------------------------------
namespace roast {
namespace {
struct MixPlan {
  std::vector<int32_t> sched;   // [pairs][len], -1 padded
  int len = 0, s1 = 2, s3 = 2;
  double makespan = 1e30, separate = 0;
};

// List-scheduling simulation of the four problems on `npairs` CTA pairs, in units of one WM = 2
// DX k-block (1024 MMA clocks; a DW k-block is half of it).  P0's units go first on every pair
// (in m- or n-major order); then each pair, when free, takes the next unit of the first class in
// the priority order whose data is ready (P2: P0 tiles (mb, 0..) published; P3: the P0 tiles of
// its token range), P1 (no dependency) as filler, else waits for the earliest ready one.
// Dependent units stream their K loop behind the P0 tiles they read.
// deterministic mode: makespan cost of one more DW split, in DX k-block units (the reduce of the
// two modules' workspaces reads every split's partial of every covering tile: ~9 us per split at
// C2, ~0.8 us per k-block).  ROAST_DET_SPLIT_COST overrides (planner experiments).
double det_split_cost() {
  const char* e = getenv("ROAST_DET_SPLIT_COST");
  return e ? atof(e) : 11.0;
}

MixPlan plan_mix(int mt0, int nt0, int kb0, int mt1, int nt1, int kbT, int mt2, int nt2, int kb2, int mt3, int nt3,
                 int npairs, double split_cost) {
  // cost model in DX k-block units: a DW k-block has half the MMA work but needs 64 B/clk of
  // operands (DX: 47), so it costs DWK = 0.6, not 0.5 (C2 fused backward 120.8 -> 118.8 us; 0.6 -
  // 0.7 give the same schedule); a unit's drain EPI_*.  ROAST_MIX_{DWK,EPI_DX,EPI_DW} override.
  auto envd = [](const char* k, double d) { const char* e = getenv(k); return e ? atof(e) : d; };
  const double EPI_DX = envd("ROAST_MIX_EPI_DX", 3.0), EPI_DW = envd("ROAST_MIX_EPI_DW", 1.0), LAT = 1.0;
  const double DWK = envd("ROAST_MIX_DWK", 0.6) * MIX_DWBK / 64.0;   // per DW k-block of MIX_DWBK tokens
  MixPlan best;
  const int units0 = mt0 * nt0;
  for (int s : {1, 2, 3, 4}) {
    const int kps = (kbT + s - 1) / s;
    const int sp = (kbT + kps - 1) / kps;
    const int units1 = mt1 * nt1 * sp, units3 = mt3 * nt3 * sp, units2 = mt2 * nt2;
    for (int order = 0; order < 2; ++order)
      for (int prio = 0; prio < 3; ++prio) {
        std::vector<double> free_t(npairs, 0.0), fin0(units0, 0.0);
        std::vector<std::vector<int32_t>> lists(npairs);
        auto pick = [&]() { return int(std::min_element(free_t.begin(), free_t.end()) - free_t.begin()); };
        for (int i = 0; i < units0; ++i) {
          const int u = order == 0 ? i : (i % mt0) * nt0 + i / mt0;
          const int q = pick();
          fin0[u] = free_t[q] + kb0 + EPI_DX;
          free_t[q] = fin0[u];
          lists[q].push_back(u);
        }
        // dependent units: ready time of their first k-block group, and finish time from a start
        auto p2_ready = [&](int u) { return fin0[(u / nt2) * nt0] + LAT; };
        auto p2_finish = [&](int u, double t) {
          const int mb = u / nt2;
          for (int g = 0; g < nt0; ++g) t = std::max(t, fin0[mb * nt0 + g] + LAT) + double(kb2) / nt0;
          return t + EPI_DX;
        };
        auto p3_range = [&](int u, int& k0, int& k1, int& nb) {
          const int split = u / (mt3 * nt3), r = u % (mt3 * nt3);
          nb = r % nt3;
          k0 = split * kps;
          k1 = std::min(k0 + kps, kbT);
        };
        // a DW k-block k of P3 reads dY_a tokens [k MIX_DWBK, (k + 1) MIX_DWBK): P0 m-blocks of 512
        auto mblk = [&](int64_t tok) { return std::min(int(tok >> 9), mt0 - 1); };
        auto p3_ready = [&](int u) {
          int k0, k1, nb;
          p3_range(u, k0, k1, nb);
          return fin0[mblk(int64_t(k0) * MIX_DWBK) * nt0 + nb] + LAT;
        };
        auto p3_finish = [&](int u, double t) {
          int k0, k1, nb;
          p3_range(u, k0, k1, nb);
          for (int k = k0; k < k1; ++k) {
            double ready = 0;
            for (int m = mblk(int64_t(k) * MIX_DWBK); m <= mblk(int64_t(k) * MIX_DWBK + MIX_DWBK - 1); ++m)
              ready = std::max(ready, fin0[m * nt0 + nb] + LAT);
            t = std::max(t, ready) + DWK;
          }
          return t + EPI_DW;
        };
        // P3 units in token order (earliest-ready first), P2 in m order, P1 as given
        std::vector<int> q1(units1), q2(units2), q3(units3);
        for (int i = 0; i < units1; ++i) q1[i] = i;
        for (int i = 0; i < units2; ++i) q2[i] = i;
        for (int i = 0; i < units3; ++i) q3[i] = i;
        std::stable_sort(q3.begin(), q3.end(), [&](int a, int b) { return p3_ready(a) < p3_ready(b); });
        size_t i1 = 0, i2 = 0, i3 = 0;
        const int classes[3][3] = {{2, 3, 1}, {3, 2, 1}, {2, 1, 3}};
        while (i1 < q1.size() || i2 < q2.size() || i3 < q3.size()) {
          const int q = pick();
          const double now = free_t[q];
          int cls = -1;
          for (int c : classes[prio]) {
            if (c == 1 && i1 < q1.size()) { cls = 1; break; }
            if (c == 2 && i2 < q2.size() && p2_ready(q2[i2]) <= now + 2.0) { cls = 2; break; }
            if (c == 3 && i3 < q3.size() && p3_ready(q3[i3]) <= now + 2.0) { cls = 3; break; }
          }
          if (cls < 0) {   // nothing ready and no filler left: the earliest-ready dependent unit
            const double r2 = i2 < q2.size() ? p2_ready(q2[i2]) : 1e30, r3 = i3 < q3.size() ? p3_ready(q3[i3]) : 1e30;
            cls = r2 <= r3 ? 2 : 3;
          }
          if (cls == 1) {
            free_t[q] = now + DWK * kps + EPI_DW;
            lists[q].push_back((1 << 24) | q1[i1++]);
          } else if (cls == 2) {
            free_t[q] = p2_finish(q2[i2], now);
            lists[q].push_back((2 << 24) | q2[i2++]);
          } else {
            free_t[q] = p3_finish(q3[i3], now);
            lists[q].push_back((3 << 24) | q3[i3++]);
          }
        }
        // deterministic mode: the fixed-order reduce after the launch reads sp partials per slot
        const double mk = *std::max_element(free_t.begin(), free_t.end()) + split_cost * sp;
        if (mk < best.makespan - 1e-9) {
          best.makespan = mk;
          best.s1 = best.s3 = sp;
          best.len = 0;
          for (auto& l : lists) best.len = std::max<int>(best.len, int(l.size()));
          best.sched.assign(size_t(npairs) * best.len, -1);
          for (int q = 0; q < npairs; ++q)
            for (size_t i = 0; i < lists[q].size(); ++i) best.sched[size_t(q) * best.len + i] = lists[q][i];
        }
      }
  }
  return best;
}

// One linear's backward, dX and dM, as one launch (roast_linear_bwd_fused): P0 = the dX units
// (512 x 256, kbx k-blocks), P1 = the dM units (256 x 256 per split, kbT DW k-blocks of MIX_DWBK
// tokens), no dependency between them.  Longest-first list scheduling over the pairs for each
// split count 1-8; `separate` = the two launches' own quantised makespans back to back (dX, then dM
// at its best split), for the caller's fused-or-not decision.  Same cost units as plan_mix.
MixPlan plan_mix1(int mtx, int ntx, int kbx, int mtw, int ntw, int kbT, int npairs) {
  auto envd = [](const char* k, double d) { const char* e = getenv(k); return e ? atof(e) : d; };
  const double EPI_DX = envd("ROAST_MIX_EPI_DX", 3.0), EPI_DW = envd("ROAST_MIX_EPI_DW", 1.0);
  const double DWK = envd("ROAST_MIX_DWK", 0.6) * MIX_DWBK / 64.0;
  const int ux = mtx * ntx;
  const double cx = kbx + EPI_DX;
  MixPlan best;
  double dw_alone = 1e30;
  for (int sp0 = 1; sp0 <= 8; ++sp0) {
    const int kps = (kbT + sp0 - 1) / sp0;
    const int sp = (kbT + kps - 1) / kps;
    const int uw = mtw * ntw * sp;
    const double cw = DWK * kps + EPI_DW;
    dw_alone = std::min(dw_alone, double((uw + npairs - 1) / npairs) * cw);
    std::vector<double> free_t(npairs, 0.0);
    std::vector<std::vector<int32_t>> lists(npairs);
    auto pick = [&]() { return int(std::min_element(free_t.begin(), free_t.end()) - free_t.begin()); };
    for (int u = 0; u < ux; ++u) {   // the longer units first
      const int q = pick();
      free_t[q] += cx;
      lists[q].push_back(u);
    }
    for (int u = 0; u < uw; ++u) {
      const int q = pick();
      free_t[q] += cw;
      lists[q].push_back((1 << 24) | u);
    }
    const double mk = *std::max_element(free_t.begin(), free_t.end());
    if (mk < best.makespan - 1e-9) {
      best.makespan = mk;
      best.s1 = sp;
      best.len = 0;
      for (auto& l : lists) best.len = std::max<int>(best.len, int(l.size()));
      best.sched.assign(size_t(npairs) * best.len, -1);
      for (int q = 0; q < npairs; ++q)
        for (size_t i = 0; i < lists[q].size(); ++i) best.sched[size_t(q) * best.len + i] = lists[q][i];
    }
  }
  best.separate = double((ux + npairs - 1) / npairs) * cx + dw_alone;
  return best;
}
}  // namespace

// dM += sum of the fused backward's dM replicas, replicas zeroed: atomic exchange / add, so a
// fold never loses a concurrent launch's reduce-adds (that launch's own fold picks them up)
__global__ void fold_dm_replicas_kernel(float* __restrict__ dM, float* __restrict__ rep, int64_t n, int reps,
                                        int64_t stride) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) acc += atomicExch(rep + r * stride + i, 0.f);
    if (acc != 0.f) atomicAdd(dM + i, acc);
  }
}

// replicas at tiny |M| only: at C2 1000x (|M| = 4720, 19 KB of dM) every weight-gradient tile of
// the fused backward reduce-adds into the same few L2 lines (131 vs 123 us at 100x); ROAST_DM_REPS
// overrides (1 = off)
static int dm_replicas(const Ctx* c) {
  if (const char* e = getenv("ROAST_DM_REPS")) return std::max(1, std::min(74, atoi(e)));
  return c->mem_size * int64_t(sizeof(float)) <= (int64_t(64) << 10) ? 16 : 1;
}

// The launch shared by the fused backwards (roast_mix_sm100): shadow / dM views (dM replicas in
// fast mode at tiny |M|), ready counters, the launch with PDL, and the replica fold after it.
// `prof` (ROAST_PROF) receives the per-CTA counters.
static long long* mix_prof = nullptr;
static roast_status_t mix_launch(Ctx* c, MixMaps& maps, MixParams& mp, const int32_t* sched, int sched_len, bool det,
                                 int pairs, cudaStream_t s) {
  roast_status_t st = ROAST_OK;
  long long*& prof = mix_prof;
  mp.neg_row = c->neg_base / 64;
  mp.reps = c->shadow_reps;
  mp.rep_rows = int(c->shadow_elems / 64);
  mp.sched = sched;
  mp.sched_len = sched_len;
  mp.err = c->d_err;
  if (const char* e = getenv("ROAST_EXP")) mp.exp = atoi(e);
  maps.shadow = *reinterpret_cast<const WMaps*>(c->tmap_shadow);
  WMaps& dmaps = *reinterpret_cast<WMaps*>(c->tmap_dm);
  if (c->tmap_dm_for != c->dM) {   // dM as 8 fp32 phase views (cached until dM is rebound)
    for (int r = 0; r < 8; ++r) {
      const int64_t elems = c->mem_size - 8 * r;
      st = make_map_2d(&dmaps.m[r], c->dM + 8 * r, 64, uint64_t(elems / 64), 256, 32, 32, true);
      if (st) return st;
    }
    c->tmap_dm_for = c->dM;
  }
  maps.dm = dmaps;
  mp.dm_reps = 1;
  mp.dm_rep_rows = 0;
  if (!det) {
    if (c->dm_reps == 0) c->dm_reps = dm_replicas(c);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (c->dm_reps > 1 && !c->dm_rep && cudaStreamIsCapturing(s, &cs) == cudaSuccess &&
        cs == cudaStreamCaptureStatusNone) {   // allocated on an eager call (not under capture)
      c->dm_rep_elems = (c->mem_size + 63) / 64 * 64;
      const size_t bytes = size_t(c->dm_reps) * size_t(c->dm_rep_elems) * sizeof(float);
      ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->dm_rep), bytes));
      ROAST_CUDA_CHECK(cudaMemsetAsync(c->dm_rep, 0, bytes, s));
      WMaps& rm = *reinterpret_cast<WMaps*>(c->tmap_dmrep);
      for (int r = 0; r < 8; ++r) {
        const int64_t elems = int64_t(c->dm_reps) * c->dm_rep_elems - 8 * r;
        if ((st = make_map_2d(&rm.m[r], c->dm_rep + 8 * r, 64, uint64_t(elems / 64), 256, 32, 32, true))) return st;
      }
    }
    if (c->dm_reps > 1 && c->dm_rep) {
      maps.dm = *reinterpret_cast<const WMaps*>(c->tmap_dmrep);
      mp.dm_reps = c->dm_reps;
      mp.dm_rep_rows = int(c->dm_rep_elems / 64);
    }
  }
  // ready counters of P0's units: the next slot of the chain ring (as sm100_chain)
  const int64_t need = std::max(1, mp.p[0].units);
  if (c->chain_slot_n < need) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return ROAST_ERR_UNSUPPORTED;
    ROAST_CUDA_CHECK(cudaDeviceSynchronize());
    cudaFree(c->chain_flags);
    c->chain_flags = nullptr;
    c->chain_slot_n = 0;
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->chain_flags), size_t(kChainSlots) * need * sizeof(int)));
    c->chain_slot_n = need;
  }
  mp.flags = c->chain_flags + int64_t(c->chain_next++ % kChainSlots) * c->chain_slot_n;
  ROAST_CUDA_CHECK(cudaMemsetAsync(mp.flags, 0, size_t(need) * sizeof(int), s));
  static std::atomic<unsigned long long> attr{0};   // smem opt-in, once per device
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(roast_mix_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, MIX_SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(mix smem)");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(pairs * 2));
  cfg.blockDim = dim3(MIX_THREADS);
  cfg.dynamicSmemBytes = MIX_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = !(getenv("ROAST_PDL") && atoi(getenv("ROAST_PDL")) == 0);
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  if (getenv("ROAST_PROF")) {   // debug: per-role wait counters, printed after a synchronising launch
    if (!prof) cudaMallocManaged(&prof, sizeof(long long) * 8 * 512);
    cudaMemset(prof, 0, sizeof(long long) * 8 * 512);
    mp.prof = prof;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, roast_mix_sm100, maps, mp);
  if (e != cudaSuccess) return cuda_fail(e, "roast_mix_sm100 launch");
  if (mp.dm_reps > 1) {
    const int64_t n = c->mem_size;
    fold_dm_replicas_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 1184)), 256, 0, s>>>(
        c->dM, c->dm_rep, n, mp.dm_reps, c->dm_rep_elems);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "fold dM replicas");
    c->launches += 1;
  }
  return ROAST_OK;
}

roast_status_t sm100_bwd_chain(Ctx* c, const Module& ma, const Module& mbm, const void* X_a, const void* Y_a,
                               const void* dY_b, void* dY_a, void* dX_a, int64_t T, cudaStream_t s, int act,
                               const void* U) {
  using namespace sm100;
  if (!supported(c, ma) || !supported(c, mbm) || cta_group() != 2 || T <= 0 || T >= (int64_t(1) << 31) ||
      getenv("ROAST_NO_BWD_FUSE"))
    return ROAST_ERR_UNSUPPORTED;
  const bool det = c->cfg.deterministic != 0;
  if (ma.H % 256 || ma.O % 256 || mbm.O % 256 || mbm.H != ma.O || !dX_a) return ROAST_ERR_UNSUPPORTED;
  const int pairs = num_sms() / 2;
  const int mtT = int((T + 511) / 512), kbT = int((T + MIX_DWBK - 1) / MIX_DWBK);   // DW k-blocks of MIX_DWBK tokens
  const std::array<int64_t, 6> key{det ? 3 : 2, ma.H, ma.O, mbm.H, mbm.O, T};   // det plans differ (split cost)
  auto it = c->chain_plans.find(key);
  auto& splits = c->mix_splits;   // plan key -> (s1, s3)
  if (it == c->chain_plans.end()) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return ROAST_ERR_UNSUPPORTED;   // planning allocates: plan on an eager call first
    bool resident = false;
    {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(unsigned(2 * pairs));
      q.blockDim = dim3(MIX_THREADS);
      q.dynamicSmemBytes = MIX_SMEM;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 2;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      q.attrs = a;
      q.numAttrs = 1;
      int ncl = 0;
      if (cudaFuncSetAttribute(roast_mix_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, MIX_SMEM) == cudaSuccess &&
          cudaOccupancyMaxActiveClusters(&ncl, roast_mix_sm100, &q) == cudaSuccess)
        resident = ncl >= pairs;
      cudaGetLastError();
    }
    MixPlan plan = plan_mix(mtT, int(mbm.H / 256), int(mbm.O / BK), int(mbm.H / 256), int(mbm.O / 256), kbT, mtT,
                            int(ma.H / 256), int(ma.O / BK), int(ma.H / 256), int(ma.O / 256), pairs,
                            det ? det_split_cost() : 0.0);
    int32_t* d = nullptr;
    if (resident) {
      ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&d), plan.sched.size() * sizeof(int32_t)));
      ROAST_CUDA_CHECK(cudaMemcpy(d, plan.sched.data(), plan.sched.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    if (getenv("ROAST_VERBOSE"))
      fprintf(stderr, "[roast] bwd chain plan: makespan %.1f (k-block units), split %d, len %d, resident %d\n",
              plan.makespan, plan.s1, plan.len, int(resident));
    it = c->chain_plans.emplace(key, std::make_pair(d, plan.len)).first;
    splits[key] = {plan.s1, plan.s3};
  }
  if (!it->second.first) return ROAST_ERR_UNSUPPORTED;
  roast_status_t st = sm100_prepare(c);
  if (st) return st;
  const int s1 = splits[key].first, s3 = splits[key].second;
  MixMaps maps;
  memset(&maps, 0, sizeof(maps));
  MixParams mp;
  memset(&mp, 0, sizeof(mp));
  auto dx_prob = [&](MixProb& P, const Module& m, const void* A, void* out, int pi) -> roast_status_t {
    P.mode = DX;
    P.M = int(T);
    P.N = int(m.H);
    P.K = int(m.O);
    P.m_tiles = mtT;
    P.n_tiles = int(m.H / 256);
    P.k_blocks = int(m.O / BK);
    P.kb_per_split = P.k_blocks;
    P.units = P.m_tiles * P.n_tiles;
    P.coord = m.d_coord_yx;
    P.coord_ld = m.nx;
    P.lam = m.lam;
    P.dep = -1;
    roast_status_t r = make_map_2d(&maps.a[pi], A, uint64_t(m.O), uint64_t(T), uint64_t(m.O) * 2, BK, 256);
    if (r) return r;
    return make_map_2d(&maps.b[pi], out, uint64_t(m.H), uint64_t(T), uint64_t(m.H) * 2, 64, 32);
  };
  auto dw_prob = [&](MixProb& P, const Module& m, const void* X, const void* dY, int sp, int pi) -> roast_status_t {
    P.mode = DW;
    P.M = int(m.H);
    P.N = int(m.O);
    P.K = int(T);
    P.m_tiles = int(m.H / 256);
    P.n_tiles = int(m.O / 256);
    P.k_blocks = kbT;
    P.kb_per_split = (kbT + sp - 1) / sp;
    P.units = P.m_tiles * P.n_tiles * ((kbT + P.kb_per_split - 1) / P.kb_per_split);
    P.off = m.d_off;
    P.sgn = m.d_sgn;
    P.ny = m.ny;
    P.lam = m.lam;
    P.dep = -1;
    P.ntiles = m.nx * m.ny;
    P.ws_slot = -1;
    roast_status_t r = make_map_blocks(&maps.a[pi], X, uint64_t(m.H), uint64_t(T), MIX_DWBK, 2);
    if (r) return r;
    return make_map_blocks(&maps.b[pi], dY, uint64_t(m.O), uint64_t(T), MIX_DWBK, 2);
  };
  if ((st = dx_prob(mp.p[0], mbm, dY_b, dY_a, 0))) return st;
  if (act) {   // dY_a = (dY_b W_b^T) * act'(U): U is layer a's pre-activation, [T x a.O]
    if (!U) return ROAST_ERR_UNSUPPORTED;
    mp.p[0].act = act;
    if ((st = make_map_2d(&maps.u, U, uint64_t(mbm.H), uint64_t(T), uint64_t(mbm.H) * 2, 64, 32))) return st;
  }
  if ((st = dw_prob(mp.p[1], mbm, Y_a, dY_b, s1, 1))) return st;
  if ((st = dx_prob(mp.p[2], ma, dY_a, dX_a, 2))) return st;
  if ((st = dw_prob(mp.p[3], ma, X_a, dY_a, s3, 3))) return st;
  mp.p[0].publish = 1;
  mp.p[2].dep = 0;
  mp.p[3].dep = 0;
  // deterministic mode (R19): the DW units store their lambda g-scaled tiles into per-tile
  // workspaces (per call, stream-ordered), reduced per slot in fixed order afterwards
  Scratch ws;
  int64_t ws_rows[2] = {0, 0};
  if (det) {
    const int dwp[2] = {1, 3};
    int64_t total = 0;
    for (int k = 0; k < 2; ++k) {
      const MixProb& P = mp.p[dwp[k]];
      ws_rows[k] = int64_t(P.units / (P.m_tiles * P.n_tiles)) * P.ntiles * 64;   // splits x tiles x 64 rows
      total += ws_rows[k];
    }
    if ((st = scratch_alloc(ws, size_t(total) * 64 * sizeof(float), s))) return st;
    int64_t row = 0;
    for (int k = 0; k < 2; ++k) {
      mp.p[dwp[k]].ws_slot = k;
      st = make_map_2d(&maps.ws[k], ws.as<float>() + row * 64, 64, uint64_t(ws_rows[k]), 256, 32, 32, true);
      if (st) return st;
      row += ws_rows[k];
    }
  }
  mp.dep_n_tiles = mp.p[0].n_tiles;
  mp.dep_m_tiles = mp.p[0].m_tiles;
  if ((st = mix_launch(c, maps, mp, it->second.first, it->second.second, det, pairs, s))) return st;
  cudaError_t e = cudaSuccess;
  long long* prof = mix_prof;
  if (det) {   // fixed order: module b's slots, then module a's (each: covering tiles, then splits)
    const int sp_b = mp.p[1].units / (mp.p[1].m_tiles * mp.p[1].n_tiles);
    const int sp_a = mp.p[3].units / (mp.p[3].m_tiles * mp.p[3].n_tiles);
    if ((e = launch_det_reduce2(c, mbm, ws.as<float>(), sp_b, &ma, ws.as<float>() + ws_rows[0] * 64, sp_a, s)) !=
        cudaSuccess)
      return cuda_fail(e, "det_reduce");
    c->launches += 1;
  }
  if (mp.prof) {
    cudaDeviceSynchronize();
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long mx = 0;
    for (int i = 0; i < 2 * pairs; ++i) {
      for (int k = 0; k < 8; ++k) acc[k] += double(prof[i * 8 + k]);
      mx = std::max(mx, prof[i * 8]);
    }
    fprintf(stderr, "[roast prof] mix: total %.0f (max %lld) | MMA wait-full DX %.0f DW %.0f | "
            "wait-tmem DX %.0f DW %.0f | DX tmem->rf per unit %.0f, release %.0f (cycles, mean per CTA / per leader)\n",
            acc[0] / (2 * pairs), mx, acc[2] / pairs, acc[4] / pairs, acc[3] / pairs,
            acc[5] / pairs, acc[6] / (acc[7] > 0 ? acc[7] : 1), acc[1] / (acc[7] > 0 ? acc[7] : 1));
  }
  c->launches++;
  return ROAST_OK;
}
// roast_linear_bwd_fused: one linear's dX GEMM and dM GEMM co-scheduled in one roast_mix_sm100
// launch when the plan beats the two launches by >= 5 % (small token counts, where a 768-wide dX
// has 48 units for 74 CTA pairs), else ROAST_ERR_UNSUPPORTED (the caller runs the two calls).
// Fast mode only (deterministic mode keeps the fixed-order reduce of the separate dM launch).
roast_status_t sm100_bwd_fused1(Ctx* c, const Module& m, const void* X, const void* dY, void* dX, int64_t T,
                                cudaStream_t s) {
  using namespace sm100;
  if (!supported(c, m) || cta_group() != 2 || T <= 0 || T >= (int64_t(1) << 31) || c->cfg.deterministic || !dX ||
      getenv("ROAST_NO_BWD_FUSE"))
    return ROAST_ERR_UNSUPPORTED;
  if (m.H % 256 || m.O % 256) return ROAST_ERR_UNSUPPORTED;
  const int pairs = num_sms() / 2;
  const int mtT = int((T + 511) / 512), kbT = int((T + MIX_DWBK - 1) / MIX_DWBK);
  const std::array<int64_t, 6> key{4, m.H, m.O, 0, 0, T};   // the plan depends on the shape only
  auto it = c->chain_plans.find(key);
  auto& splits = c->mix_splits;   // plan key -> (split, unused)
  if (it == c->chain_plans.end()) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return ROAST_ERR_UNSUPPORTED;   // plan on an eager call first
    bool resident = false;
    {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(unsigned(2 * pairs));
      q.blockDim = dim3(MIX_THREADS);
      q.dynamicSmemBytes = MIX_SMEM;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 2;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      q.attrs = a;
      q.numAttrs = 1;
      int ncl = 0;
      if (cudaFuncSetAttribute(roast_mix_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, MIX_SMEM) == cudaSuccess &&
          cudaOccupancyMaxActiveClusters(&ncl, roast_mix_sm100, &q) == cudaSuccess)
        resident = ncl >= pairs;
      cudaGetLastError();
    }
    MixPlan plan = plan_mix1(mtT, int(m.H / 256), int(m.O / BK), int(m.H / 256), int(m.O / 256), kbT, pairs);
    int32_t* d = nullptr;
    const bool pays = getenv("ROAST_FUSE1_ALWAYS") != nullptr || plan.makespan < 0.95 * plan.separate;
    if (resident && pays) {
      ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&d), plan.sched.size() * sizeof(int32_t)));
      ROAST_CUDA_CHECK(cudaMemcpy(d, plan.sched.data(), plan.sched.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    if (getenv("ROAST_VERBOSE"))
      fprintf(stderr, "[roast] bwd fused1 %lld x %lld, T %lld: makespan %.1f vs separate %.1f, split %d, used %d\n",
              (long long)m.H, (long long)m.O, (long long)T, plan.makespan, plan.separate, plan.s1, int(d != nullptr));
    it = c->chain_plans.emplace(key, std::make_pair(d, plan.len)).first;
    splits[key] = {plan.s1, 0};
  }
  if (!it->second.first) return ROAST_ERR_UNSUPPORTED;
  roast_status_t st = sm100_prepare(c);
  if (st) return st;
  const int sp = splits[key].first;
  MixMaps maps;
  memset(&maps, 0, sizeof(maps));
  MixParams mp;
  memset(&mp, 0, sizeof(mp));
  MixProb& P = mp.p[0];   // dX = lambda dY W~^T
  P.mode = DX;
  P.M = int(T);
  P.N = int(m.H);
  P.K = int(m.O);
  P.m_tiles = mtT;
  P.n_tiles = int(m.H / 256);
  P.k_blocks = int(m.O / BK);
  P.kb_per_split = P.k_blocks;
  P.units = P.m_tiles * P.n_tiles;
  P.coord = m.d_coord_yx;
  P.coord_ld = m.nx;
  P.lam = m.lam;
  P.dep = -1;
  P.ws_slot = -1;
  if ((st = make_map_2d(&maps.a[0], dY, uint64_t(m.O), uint64_t(T), uint64_t(m.O) * 2, BK, 256))) return st;
  if ((st = make_map_2d(&maps.b[0], dX, uint64_t(m.H), uint64_t(T), uint64_t(m.H) * 2, 64, 32))) return st;
  MixProb& W = mp.p[1];   // dM += scatter(lambda g X^T dY)
  W.mode = DW;
  W.M = int(m.H);
  W.N = int(m.O);
  W.K = int(T);
  W.m_tiles = int(m.H / 256);
  W.n_tiles = int(m.O / 256);
  W.k_blocks = kbT;
  W.kb_per_split = (kbT + sp - 1) / sp;
  W.units = W.m_tiles * W.n_tiles * ((kbT + W.kb_per_split - 1) / W.kb_per_split);
  W.off = m.d_off;
  W.sgn = m.d_sgn;
  W.ny = m.ny;
  W.lam = m.lam;
  W.dep = -1;
  W.ntiles = m.nx * m.ny;
  W.ws_slot = -1;
  if ((st = make_map_blocks(&maps.a[1], X, uint64_t(m.H), uint64_t(T), MIX_DWBK, 2))) return st;
  if ((st = make_map_blocks(&maps.b[1], dY, uint64_t(m.O), uint64_t(T), MIX_DWBK, 2))) return st;
  for (int k = 2; k < 4; ++k) {   // unused problem slots: valid descriptors (prefetched), no units
    maps.a[k] = maps.a[0];
    maps.b[k] = maps.b[0];
    mp.p[k].ws_slot = -1;
    mp.p[k].dep = -1;
  }
  mp.dep_n_tiles = 1;
  mp.dep_m_tiles = 1;
  if ((st = mix_launch(c, maps, mp, it->second.first, it->second.second, false, pairs, s))) return st;
  c->launches++;
  return ROAST_OK;
}
}  // namespace roast
