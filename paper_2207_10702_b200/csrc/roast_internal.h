// roast_internal.h — handle state shared by the C-ABI layer and the kernels.
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <array>
#include <map>
#include <string>
#include <vector>

#include "../../include/roast.h"
#include "roast_hash.cuh"

namespace roast {

enum ModuleKind { kLinear = 0, kEmbedding = 1 };
constexpr int32_t kGroupIdBase = 1 << 24;

struct Module {
  ModuleKind kind;
  float lam;
  ModuleHash hash;
  // linear
  int64_t H = 0, O = 0;
  int32_t nx = 0, ny = 0;         // tile grid
  int64_t* d_off = nullptr;       // [nx * ny] tile offsets (elements)
  int8_t* d_sgn = nullptr;        // [nx * ny] tile signs
  std::vector<int64_t> h_off;     // host copies
  std::vector<int8_t> h_sgn;
  // deterministic reduce (K5): tiles sorted by (offset, tile id); the kernel
  // binary-searches the covering range [lo, hi) of every A-aligned slot group.
  int32_t* d_sorted = nullptr;    // [ntiles] tile ids
  int64_t* d_sorted_off = nullptr;// [ntiles]
  // deterministic mode, heavily shared memories: the covering range [lo, hi) in the sorted
  // list of every 4-slot group of M (static; built at registration when <= 64 MB), so the
  // warp-per-group reduce reads it instead of two dependent binary searches per group
  int32_t* d_cover = nullptr;     // [ceil(|M| / 4)][2]
  // tcgen05 producer: packed TMA coordinates of every tile, (off >> 6) << 4 | neg << 3 | (off >> 3) & 7,
  // in [x][y] order (FWD walks a row) and [y][x] order (DX walks a column).  Empty if off >= 2^33.
  int32_t* d_coord_xy = nullptr;
  int32_t* d_coord_yx = nullptr;
  // embedding
  int64_t rows = 0;
  int32_t dim = 0, chunk = 0, chunks_per_row = 0;
};

// one-shot P2P exchange: at most one NVSwitch domain (8 GPUs) of ranks
constexpr int kP2PMaxWorld = 8;
// window layout (bytes): [0, 128) int32 flags[world] (rank r writes flags[r] = epoch after its
// post) | [128, 256) int32 flags2[world] (two-shot: rank r's slice of M is updated) |
// [256] int32 epoch, [260] u32 arrival counter | [512, ...) buffer 0, buffer 1 (packed
// gradients) and the two-shot M buffer, p2p_n fp32 each (rounded up to 4)
constexpr int64_t kP2PHeader = 512;

struct P2PView {   // what the fused update kernel needs (kernels_simt.cu opt_kernel)
  int world = 0;
  const float* buf0[kP2PMaxWorld] = {};   // each rank's buffer 0; buffer 1 = + stride floats
  int64_t stride = 0;
  const int* flags = nullptr;             // this rank's flags[world]
  const int* epoch = nullptr;             // this rank's epoch word
  int* err = nullptr;                     // sticky device error word (timeout)
  // two-shot (reduce-scatter phase): only packed indices [lo, hi) are updated, and the new M
  // values are also written to mout[p] for the other ranks to gather
  int64_t lo = 0, hi = -1;                // hi < 0: all of [0, n)
  float* mout = nullptr;
  // NVLS: the gradient of index p is multimem.ld_reduce(mc_buf0 + parity + p) (the sum over the
  // ranks, reduced in the switch); two-shot new values go out with multimem.st to mc_mout + p
  const float* mc_buf0 = nullptr;
  float* mc_mout = nullptr;
};

#ifdef __CUDACC__
// Writers of the bf16 shadow (sync_shadow, the optimizer pass, the P2P gather) refresh every
// replica: at small |M| the shadow is kept `reps` times (rep_stride elements apart) so the
// tcgen05 GEMMs' hashed-tile loads spread over reps x more L2 lines (CTA pair p reads replica
// p % reps); 16-bit halves, V = 4 packed as uint2.
struct ShadowOut {
  unsigned short* sh;
  int64_t neg_base;
  int64_t rep_stride;
  int reps;
  __device__ __forceinline__ void store4(int64_t i, uint2 pos) const {
    const uint2 neg = make_uint2(pos.x ^ 0x80008000u, pos.y ^ 0x80008000u);   // bf16 negation = sign flip
    for (int r = 0; r < reps; ++r) {
      *reinterpret_cast<uint2*>(sh + r * rep_stride + i) = pos;
      *reinterpret_cast<uint2*>(sh + r * rep_stride + neg_base + i) = neg;
    }
  }
  __device__ __forceinline__ void store1(int64_t i, unsigned short b) const {
    for (int r = 0; r < reps; ++r) {
      sh[r * rep_stride + i] = b;
      sh[r * rep_stride + neg_base + i] = b ^ 0x8000u;
    }
  }
};

// Touched-slot traversal (exchange.cu pack, p2p.cu post, kernels_simt.cu opt_kernel): the
// packed index space [0, n) is cut into one contiguous range per CTA (threads of a CTA still
// touch consecutive vectors); a thread finds its interval once by binary search and afterwards
// only steps forward, instead of a dependent binary search per element.
struct IvWalk {
  const int64_t* start;    // interval starts in M
  const int64_t* prefix;   // exclusive prefix of interval lengths (prefix[0] = 0)
  int n_iv;
  int i = 0;
  __device__ void seek(int64_t p) {   // the largest i with prefix[i] <= p
    int lo = 0, hi = n_iv - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(prefix + mid) <= p) lo = mid; else hi = mid - 1;
    }
    i = lo;
  }
  __device__ int64_t slot(int64_t p) {   // p must not decrease between calls
    while (i + 1 < n_iv && __ldg(prefix + i + 1) <= p) ++i;
    return __ldg(start + i) + (p - __ldg(prefix + i));
  }
};

// [*b, *e): this CTA's contiguous share of [0, n), a multiple of blockDim.x * V long
__device__ inline void cta_range(int64_t n, int V, int64_t* b, int64_t* e) {
  const int64_t q = int64_t(blockDim.x) * V;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t chunk = (per + q - 1) / q * q;
  *b = int64_t(blockIdx.x) * chunk;
  *e = *b + chunk < n ? *b + chunk : n;
}
#endif

struct Ctx {
  int64_t mem_size = 0;
  uint64_t seed = 0;
  roast_tile_t tile{0, 0};
  roast_config_t cfg{};
  float* M = nullptr;
  float* dM = nullptr;
  uint16_t* shadow = nullptr;     // [2 * mem_size + pad] bf16 bits: +bf16(M) then -bf16(M)
  int64_t shadow_elems = 0;
  int64_t neg_base = 0;           // index of the negated copy (128-B aligned)
  int shadow_reps = 1;            // replicas of the shadow, shadow_elems apart (small |M|: spread L2 lines)
  std::vector<Module> modules;
  // roast_register_linear_concat: linears sharing in_features fused along out_features (their
  // tile maps side by side, one GEMM per call); ids kGroupIdBase + index, outside the module
  // id space so they never shift the hash keys of later registrations
  std::vector<Module> groups;
  int64_t identity_cursor = 0;    // IDENTITY mapping: next free base
  // device error flag (sticky)
  int32_t* d_err = nullptr;
  int64_t* d_zero_idx = nullptr;  // device int64 0 (inside the d_err block): row 0 for biases via L
  // comm
  void* nccl_comm = nullptr;
  int32_t rank = 0, world = 1;
  int64_t launches = 0;
  // tcgen05 path: cached TMA descriptors of the shadow (rebuilt on bind)
  alignas(64) unsigned char tmap_shadow[1024];
  alignas(64) unsigned char tmap_shadow_half[1024];   // the same views with 32-row boxes (DX, N per unit 192)
  bool tmap_shadow_valid = false;
  // ... and of dM (8 fp32 phase views for the TMA reduce-add epilogue), valid for dM == tmap_dm_for
  alignas(64) unsigned char tmap_dm[1024];
  const float* tmap_dm_for = nullptr;
  // dM replicas of the fused backward at tiny |M| (fast mode): its weight-gradient tiles reduce-add
  // into replica (CTA pair % dm_reps) instead of all into the same few L2 lines, and a fold adds
  // the replicas into dM (and zeroes them) after the launch; [dm_reps][dm_rep_elems] fp32
  float* dm_rep = nullptr;
  int dm_reps = 0;                // 0: not decided yet
  int64_t dm_rep_elems = 0;
  alignas(64) unsigned char tmap_dmrep[1024];
  // optimizer state, |M| fp32 each (Adagrad: s1 = G; Adam: s1 = m, s2 = v)
  float* opt_s1 = nullptr;
  float* opt_s2 = nullptr;
  // kernel-configuration autotuner (roast_set_autotune): (kernel, H, O, tokens) -> (WM, split-K)
  int autotune = 0;
  std::map<std::array<int64_t, 4>, std::pair<int, int>> tuned;
  // chained GEMM pairs (roast_linear_fwd_chain / roast_linear_bwd_dx_chain): per-shape static
  // schedules on the device (pointer, per-pair length; null = chaining does not pay) and the
  // ready counters of the first GEMM's output tiles
  std::map<std::array<int64_t, 6>, std::pair<int32_t*, int>> chain_plans;
  // ... and the fused backwards' split-K counts of their weight-gradient problems (P1, P3)
  std::map<std::array<int64_t, 6>, std::pair<int, int>> mix_splits;
  // ready counters of chained launches: kChainSlots slots of chain_slot_n ints, handed out round
  // robin per launch, so chained launches in flight on different streams use different counters
  // (up to kChainSlots launches in flight per handle); grown only outside graph capture
  int* chain_flags = nullptr;
  int64_t chain_slot_n = 0;
  uint32_t chain_next = 0;
  // touched-set dM exchange (exchange.cu): merged intervals of the slots the registered modules
  // can write; d_iv = [starts (n_iv) | exclusive prefix of lengths (n_iv + 1)], d_pack = the
  // packed buffer (touched_n fp32); rebuilt when the module count changes
  int32_t exchange_mode = 0;      // roast_exchange_mode_t
  bool touched_valid = false, touched_vec = false;
  int64_t touched_for = -1, touched_n = 0;
  int32_t n_iv = 0;
  int64_t* d_iv = nullptr;
  float* d_pack = nullptr;
  // one-shot P2P exchange (p2p.cu): this rank's window (flags | epoch | two packed buffers of
  // p2p_n fp32) and every rank's window mapped into this process (IPC or attach)
  char* p2p_win = nullptr;
  int64_t p2p_bytes = 0, p2p_n = 0;
  int32_t p2p_rank = 0, p2p_world = 0;
  char* p2p_peer[kP2PMaxWorld] = {};
  bool p2p_opened[kP2PMaxWorld] = {};
  // NVLS (nvls.cu): the window lives in driver-API memory bound to a multicast object; p2p_win
  // is then its unicast mapping and nvls_mc_va the multicast mapping of the same offsets
  unsigned long long nvls_mc = 0, nvls_phys = 0;       // CUmemGenericAllocationHandle
  unsigned long long nvls_uc_va = 0, nvls_mc_va = 0;   // CUdeviceptr
  size_t nvls_size = 0;
  int32_t nvls_world = 0, nvls_dev = -1;
  bool nvls_have_mc = false, nvls_added = false, nvls_memb = false, nvls_bound = false;
};

#ifdef __CUDACC__
inline ShadowOut shadow_out(const Ctx* c) {
  return ShadowOut{c->shadow, c->neg_base, c->shadow_elems, c->shadow_reps};
}
#endif

// error reporting (thread-local detail string)
roast_status_t fail(roast_status_t st, const std::string& msg);
roast_status_t cuda_fail(cudaError_t e, const char* what);
#define ROAST_CUDA_CHECK(call)                                   \
  do {                                                           \
    cudaError_t _e = (call);                                     \
    if (_e != cudaSuccess) return ::roast::cuda_fail(_e, #call); \
  } while (0)

void comm_destroy(Ctx* c);
void p2p_destroy(Ctx* c);   // p2p.cu: close peer mappings, free the window
void nvls_destroy(Ctx* c);  // nvls.cu: unmap and release the multicast object and its memory

// touched-set exchange (exchange.cu): build the interval tables (host, synchronous uploads);
// pack (dir 0: d_pack <- dM[touched]) or unpack (dir 1: dM[touched] <- scale * d_pack)
roast_status_t touched_prepare(Ctx* c, cudaStream_t s);
// optimizer-call validation, state allocation and (need_touched) the interval tables
roast_status_t opt_prepare(Ctx* c, const roast_opt_config_t* cfg, int64_t step, bool need_touched, cudaStream_t s);
cudaError_t launch_pack(Ctx* c, int dir, float scale, cudaStream_t s);

constexpr int kChainSlots = 64;
// Per-call scratch (deterministic dM partials, the deterministic embedding sort): allocated with cudaMallocAsync on the call's stream and freed with cudaFreeAsync on
// the same stream after the kernels that use it are enqueued, so calls on different streams never
// share scratch and graph capture records alloc / free nodes.  The device's default
// memory pool keeps freed blocks (release threshold set at roast_create), so steady-state calls
// do not go back to the driver.
// One-time per-device set-up (e.g. a kernel's shared-memory opt-in, which is per device): true
// the first time it is called for the current device with this mask (one bit per device < 64).
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned long long bit = 1ull << (d & 63);
  return !(mask.fetch_or(bit) & bit);
}

struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() { if (p) cudaFreeAsync(p, s); }
  template <class T> T* as() const { return static_cast<T*>(p); }
};
roast_status_t scratch_alloc(Scratch& w, size_t bytes, cudaStream_t s);

// ---- kernel launchers (return cudaError_t of the launch) ----------------------
// SIMT paths (any tile geometry), T = float or bf16 storage selected by dt
cudaError_t launch_simt_fwd(const Ctx* c, const Module& m, const void* X, void* Y, int64_t T, roast_dtype_t dt,
                            bool transpose_w, cudaStream_t s, const float* bias = nullptr);
// bias backward, first half: db[j] = sum_t dY[t, j] in fp32, fixed order (slab partials
// then an in-order sum over slabs) -> db [n]
cudaError_t launch_colsum(const void* dY, int64_t T, int n, int64_t ld, roast_dtype_t dt, float* partial, float* db,
                          cudaStream_t s, int accumulate = 0);
int colsum_slabs(int64_t T, int n);
cudaError_t launch_simt_dw(const Ctx* c, const Module& m, const void* X, const void* dY, int64_t T,
                           roast_dtype_t dt, float* ws, cudaStream_t s);
cudaError_t launch_det_reduce(Ctx* c, const Module& m, const float* ws, int nsplit, cudaStream_t s);
// two modules' workspaces into dM in one launch: the result of launch_det_reduce(m0) then (m1)
cudaError_t launch_det_reduce2(Ctx* c, const Module& m0, const float* ws0, int ns0, const Module* m1,
                               const float* ws1, int ns1, cudaStream_t s);
cudaError_t launch_sync_shadow(Ctx* c, cudaStream_t s);
cudaError_t launch_optimizer(Ctx* c, int kind, float lr, float b1, float b2, float eps, float wd, int64_t step,
                             int zero, bool touched_only, cudaStream_t s, const float* gpack = nullptr,
                             const P2PView* p2p = nullptr);
cudaError_t launch_materialize(const Ctx* c, const Module& m, roast_dtype_t dt, void* W, cudaStream_t s);
cudaError_t launch_embed_fwd(const Ctx* c, const Module& m, const int64_t* idx, int64_t n, float* out,
                             cudaStream_t s);
cudaError_t launch_embed_bwd(const Ctx* c, const Module& m, const int64_t* idx, int64_t n, const float* dOut,
                             cudaStream_t s);
constexpr int kEmbMaxTables = 64;  // tables per fused launch (kernel-parameter budget)
// nt <= kEmbMaxTables tables of equal dim / chunk; idx / out / dOut are table-major
// (nt x n rows); dOut == nullptr selects the forward
cudaError_t launch_embed_multi(const Ctx* c, const Module* const* mods, int nt, const int64_t* idx, int64_t n,
                               float* out, const float* dOut, cudaStream_t s);
cudaError_t launch_chunk_map(const Ctx* c, const Module& m, const int64_t* rows, int64_t n, int64_t* off,
                             int8_t* sgn, cudaStream_t s);

// tcgen05 paths (bf16, Z1 = Z2 = 64)
// deterministic embedding backward: key by offset, stable radix sort, fixed-order per-slot sum
roast_status_t embed_bwd_deterministic(Ctx* c, const Module* const* mods, int nt, const int64_t* idx, int64_t n,
                                       const float* dOut, cudaStream_t s);
roast_status_t sm100_prepare(Ctx* c);  // build shadow tensor map
roast_status_t sm100_fwd(Ctx* c, const Module& m, const void* X, void* Y, int64_t T, const float* bias,
                         cudaStream_t s);
// two dependent GEMMs in one persistent launch: FWD Y_a = X W_a, Y_b = Y_a W_b (dx = false) or
// DX dY_a = dY_b W_b^T, dX = dY_a W_a^T (dx = true; m0 = the layer whose dX is computed first).
// Returns ROAST_ERR_UNSUPPORTED when the shapes are not on the tcgen05 path or chaining would
// not beat two launches (the caller then makes two launches).
roast_status_t sm100_chain(Ctx* c, const Module& m0, const Module& m1, const void* A0, void* out0, void* out1,
                           int64_t T, bool dx, const float* bias0, const float* bias1, cudaStream_t s, int act = 0,
                           void* act_buf = nullptr);
roast_status_t sm100_dx(Ctx* c, const Module& m, const void* dY, void* dX, int64_t T, cudaStream_t s);
// the same with an activation fused into the register-held epilogue (roast_linear_fwd_act / _bwd_dx_act)
roast_status_t sm100_fwd_act(Ctx* c, const Module& m, const void* X, void* Y, void* A, int64_t T, const float* bias,
                             int act, cudaStream_t s);
roast_status_t sm100_dx_act(Ctx* c, const Module& m, const void* dY, const void* U, void* dX, int64_t T, int act,
                            cudaStream_t s);
// the whole backward of a chained pair a -> b (Y_a = X_a W_a, Y_b = Y_a W_b) in one persistent
// launch: dY_a = dY_b W_b^T, dM += b(Y_a, dY_b), dX_a = dY_a W_a^T, dM += a(X_a, dY_a), the four
// GEMMs co-scheduled (gemm_sm100.cu roast_mix_sm100).  ROAST_ERR_UNSUPPORTED when the shapes /
// mode do not allow it (the caller then makes the four launches).
// one linear's dX and dM GEMMs co-scheduled in one launch (small token counts); UNSUPPORTED when
// the plan does not beat the two launches, the geometry is not 256-aligned, or in deterministic mode
roast_status_t sm100_bwd_fused1(Ctx* c, const Module& m, const void* X, const void* dY, void* dX, int64_t T,
                                cudaStream_t s);
roast_status_t sm100_bwd_chain(Ctx* c, const Module& ma, const Module& mb, const void* X_a, const void* Y_a,
                               const void* dY_b, void* dY_a, void* dX_a, int64_t T, cudaStream_t s, int act = 0,
                               const void* U = nullptr);
roast_status_t sm100_dw(Ctx* c, const Module& m, const void* X, const void* dY, int64_t T, cudaStream_t s);

}  // namespace roast
