// One-shot P2P dM exchange fused with the update (the exchange is
// a6 = P:194, the update a7 = P:440 / P:749-813).
//
// NCCL's all-reduce and the optimizer pass are two launches with a full HBM round trip of
// the packed gradient between them (roast_grad_exchange_step).  Here every rank maps every
// other rank's exchange window (CUDA IPC over NVLink / NVSwitch, or plain pointers for ranks
// that share a process) and the update kernel reads the W packed gradients straight from the
// peers' HBM, sums them in rank order (so every rank computes bit-identical sums and M stays
// replicated without a broadcast) and applies the optimizer, the shadow refresh and the dM
// zeroing in the same pass.  Per step and rank: one post launch (dM touched slots -> own
// buffer, then a flag store to every peer) and one update launch.
//
// Synchronisation is stream-ordered and graph-capturable: the epoch lives in device memory.
//   post   : e = epoch + 1; pack into buffer (e & 1); the last CTA: fence, flags_r[rank] = e on
//            every rank r (st.release.sys), epoch = e
//   finish : every CTA waits for flags[r] >= e for all r (ld.acquire.sys), then reads buffer
//            (e & 1) of every rank
// Two buffers make the reuse safe: a rank writes buffer (e & 1) again at epoch e + 2 only after
// its own finish(e + 1), which waited for every peer's post(e + 1), which each peer issued
// after its finish(e) had stopped reading that buffer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <type_traits>

#include "roast_internal.h"

namespace roast {
namespace {

struct PeerWins {
  char* w[kP2PMaxWorld];
};

// buffer (epoch + 1) & 1 of this rank's window <- dM at the touched slots; the last CTA to
// finish publishes the new epoch in every rank's flags[rank] (release, system scope) and
// advances the local epoch.  Every CTA read the epoch before it arrived at the counter, so the
// update cannot change the buffer any CTA chose.  Peers read this window through this GPU's
// L2, so a GPU-scope fence per CTA orders the packed data before the flag.
// NVLS (mc_flags = the multicast alias of the flags array): one multimem.st writes flags[rank] on
// every rank, after fence.proxy.alias orders the unicast packing before the peers' multicast reads.
__device__ __forceinline__ void nvls_signal(int* mc_flag, int e) {
  asm volatile("fence.proxy.alias;" ::: "memory");
  __threadfence_system();
  asm volatile("multimem.st.release.sys.global.b32 [%0], %1;" ::"l"(mc_flag), "r"(e) : "memory");
}

template <int V>
__global__ void p2p_post_kernel(const float* __restrict__ dM, PeerWins peers, int world, int rank, int64_t stride,
                                const int64_t* __restrict__ start, const int64_t* __restrict__ prefix, int n_iv,
                                int64_t total, int* mc_flags) {
  using VT = typename std::conditional<V == 4, float4, float>::type;
  char* win = peers.w[rank];
  int* epoch = reinterpret_cast<int*>(win + 256);
  unsigned* arrived = reinterpret_cast<unsigned*>(win + 260);
  const int e = *reinterpret_cast<const volatile int*>(epoch) + 1;
  float* buf = reinterpret_cast<float*>(win + kP2PHeader) + ((e & 1) ? stride : 0);
  int64_t b, end;
  cta_range(total, V, &b, &end);
  IvWalk w{start, prefix, n_iv};
  if (b + int64_t(threadIdx.x) * V < end) w.seek(b + int64_t(threadIdx.x) * V);
  for (int64_t p = b + int64_t(threadIdx.x) * V; p < end; p += int64_t(blockDim.x) * V)
    *reinterpret_cast<VT*>(buf + p) = *reinterpret_cast<const VT*>(dM + w.slot(p));
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(arrived, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (mc_flags) {
    if (threadIdx.x == 0) nvls_signal(mc_flags + rank, e);
  } else if (threadIdx.x < world) {
    int* f = reinterpret_cast<int*>(peers.w[threadIdx.x]) + rank;
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(f), "r"(e) : "memory");
  }
  if (threadIdx.x == 0) {
    *reinterpret_cast<volatile int*>(epoch) = e;
    *reinterpret_cast<volatile unsigned*>(arrived) = 0u;
  }
}

// two-shot: after this rank's slice of M is updated (and copied to its M buffer), publish the
// current epoch in every rank's flags2[rank]
__global__ void p2p_signal2_kernel(PeerWins peers, int world, int rank, int* mc_flags2) {
  const int e = *reinterpret_cast<const volatile int*>(peers.w[rank] + 256);
  __threadfence();
  if (mc_flags2) {
    if (threadIdx.x == 0) nvls_signal(mc_flags2 + rank, e);
  } else if (threadIdx.x < world) {
    int* f = reinterpret_cast<int*>(peers.w[threadIdx.x] + 128) + rank;
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(f), "r"(e) : "memory");
  }
}

struct Slices {   // packed-index slice [at[r], at[r + 1]) is updated by rank r
  int64_t at[kP2PMaxWorld + 1];
};

// two-shot gather: wait until every rank has published its slice (flags2 >= epoch), then copy
// the other ranks' new values into M at the touched slots, refresh both shadow halves, zero dM
template <int V>
__global__ void p2p_gather_kernel(float* __restrict__ M, float* __restrict__ dM, ShadowOut so, PeerWins peers, int world, int rank, Slices sl, int64_t stride,
                                  const int64_t* __restrict__ start, const int64_t* __restrict__ prefix, int n_iv,
                                  int64_t n, int* err) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    const char* win = peers.w[rank];
    const int e = *reinterpret_cast<const volatile int*>(win + 256);
    const int* f2 = reinterpret_cast<const int*>(win + 128);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < world; ++r) {
      int f;
      for (;;) {
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(f) : "l"(f2 + r) : "memory");
        if (f - e >= 0) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {
          atomicOr(err, 2);
          __threadfence_system();
          __trap();
        }
        __nanosleep(64);
      }
    }
    s_ok = 1;
    asm volatile("fence.proxy.alias;" ::: "memory");   // NVLS: mout arrived through the multicast alias
  }
  __syncthreads();
  using VT = typename std::conditional<V == 4, float4, float>::type;
  int64_t b, end;
  cta_range(n, V, &b, &end);
  IvWalk w{start, prefix, n_iv};
  if (b + int64_t(threadIdx.x) * V < end) w.seek(b + int64_t(threadIdx.x) * V);
  int owner = 0;
  for (int64_t p = b + int64_t(threadIdx.x) * V; p < end; p += int64_t(blockDim.x) * V) {
    const int64_t i = w.slot(p);
    while (owner + 1 < world && sl.at[owner + 1] <= p) ++owner;
    if (owner == rank) continue;   // updated in place by this rank's reduce phase
    const float* src = reinterpret_cast<const float*>(peers.w[owner] + kP2PHeader) + 2 * stride + p;
    const VT v = __ldcv(reinterpret_cast<const VT*>(src));
    *reinterpret_cast<VT*>(M + i) = v;
    if constexpr (V == 4) {
      const __nv_bfloat162 p0 = __floats2bfloat162_rn(v.x, v.y), p1 = __floats2bfloat162_rn(v.z, v.w);
      uint2 pos;
      pos.x = *reinterpret_cast<const uint32_t*>(&p0);
      pos.y = *reinterpret_cast<const uint32_t*>(&p1);
      so.store4(i, pos);
      *reinterpret_cast<float4*>(dM + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      so.store1(i, __bfloat16_as_ushort(__float2bfloat16_rn(v)));
      dM[i] = 0.f;
    }
  }
  (void)s_ok;
}

}  // namespace
}  // namespace roast

using namespace roast;

namespace {

Ctx* pctx(roast_t h) { return reinterpret_cast<Ctx*>(h); }

void p2p_release(Ctx* c) {
  for (int r = 0; r < kP2PMaxWorld; ++r) {
    if (c->p2p_opened[r] && c->p2p_peer[r]) cudaIpcCloseMemHandle(c->p2p_peer[r]);
    c->p2p_opened[r] = false;
    c->p2p_peer[r] = nullptr;
  }
  c->p2p_world = 0;
}

// the window's multicast alias at byte offset off (NVLS bound), else null
int* mc_int(const Ctx* c, int64_t off) {
  return c->nvls_bound ? reinterpret_cast<int*>(c->nvls_mc_va + off) : nullptr;
}

bool p2p_ready(const Ctx* c) {
  return c->p2p_world > 0 && c->p2p_win && c->touched_valid && c->touched_for == int64_t(c->modules.size()) &&
         c->touched_n == c->p2p_n;
}

}  // namespace

namespace roast {
void p2p_destroy(Ctx* c) {
  p2p_release(c);
  if (c->nvls_bound) c->p2p_win = nullptr;   // the window is the NVLS unicast mapping: nvls_destroy unmaps it
  nvls_destroy(c);
  cudaFree(c->p2p_win);
  c->p2p_win = nullptr;
  c->p2p_bytes = c->p2p_n = 0;
}
}  // namespace roast

extern "C" {

roast_status_t roast_p2p_window(roast_t h, void** window, int64_t* bytes) {
  Ctx* c = pctx(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  if (roast_status_t st = touched_prepare(c, 0)) return st;
  if (c->nvls_bound) {   // the NVLS window was sized for this touched set at roast_nvls_bind
    if (c->p2p_n != c->touched_n) return fail(ROAST_ERR_STATE, "NVLS window bound before the last registration");
    if (window) *window = c->p2p_win;
    if (bytes) *bytes = c->p2p_bytes;
    return ROAST_OK;
  }
  const int64_t n = (c->touched_n + 3) / 4 * 4;   // keep buffer 1 16-byte aligned
  const int64_t need = kP2PHeader + 3 * n * int64_t(sizeof(float));   // 2 gradient buffers + M buffer
  if (!c->p2p_win || c->p2p_n != c->touched_n) {
    p2p_release(c);
    cudaFree(c->p2p_win);
    c->p2p_win = nullptr;
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->p2p_win), size_t(need)));
    ROAST_CUDA_CHECK(cudaMemset(c->p2p_win, 0, size_t(need)));   // flags and epoch start at 0 on every rank
    c->p2p_bytes = need;
    c->p2p_n = c->touched_n;
  }
  if (window) *window = c->p2p_win;
  if (bytes) *bytes = c->p2p_bytes;
  return ROAST_OK;
}

roast_status_t roast_p2p_ipc_handle(roast_t h, uint8_t handle[64]) {
  Ctx* c = pctx(h);
  if (!handle) return fail(ROAST_ERR_CONFIG, "null handle buffer");
  if (roast_status_t st = roast_p2p_window(h, nullptr, nullptr)) return st;
  cudaIpcMemHandle_t ipc;
  ROAST_CUDA_CHECK(cudaIpcGetMemHandle(&ipc, c->p2p_win));
  static_assert(sizeof(ipc) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &ipc, 64);
  return ROAST_OK;
}

roast_status_t roast_p2p_attach(roast_t h, int32_t rank, int32_t world, void* const* windows) {
  Ctx* c = pctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (c->nvls_bound) return fail(ROAST_ERR_STATE, "p2p: this handle's window is bound to an NVLS multicast object");
  if (world < 1 || world > kP2PMaxWorld || rank < 0 || rank >= world || !windows)
    return fail(ROAST_ERR_CONFIG, "p2p: 1 <= world <= 8, 0 <= rank < world, windows[world]");
  if (roast_status_t st = roast_p2p_window(h, nullptr, nullptr)) return st;
  if (windows[rank] != c->p2p_win) return fail(ROAST_ERR_CONFIG, "p2p: windows[rank] must be this handle's window");
  p2p_release(c);
  for (int r = 0; r < world; ++r) c->p2p_peer[r] = static_cast<char*>(windows[r]);
  c->p2p_rank = rank;
  c->p2p_world = world;
  return ROAST_OK;
}

roast_status_t roast_p2p_open(roast_t h, int32_t rank, int32_t world, const uint8_t* handles) {
  Ctx* c = pctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (c->nvls_bound) return fail(ROAST_ERR_STATE, "p2p: this handle's window is bound to an NVLS multicast object");
  if (world < 1 || world > kP2PMaxWorld || rank < 0 || rank >= world || !handles)
    return fail(ROAST_ERR_CONFIG, "p2p: 1 <= world <= 8, 0 <= rank < world, handles[world * 64]");
  if (roast_status_t st = roast_p2p_window(h, nullptr, nullptr)) return st;
  p2p_release(c);
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      c->p2p_peer[r] = c->p2p_win;
      continue;
    }
    cudaIpcMemHandle_t ipc;
    memcpy(&ipc, handles + size_t(r) * 64, 64);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      p2p_release(c);
      return cuda_fail(e, "cudaIpcOpenMemHandle");
    }
    c->p2p_peer[r] = static_cast<char*>(p);
    c->p2p_opened[r] = true;
  }
  c->p2p_rank = rank;
  c->p2p_world = world;
  return ROAST_OK;
}

roast_status_t roast_p2p_post(roast_t h, roast_stream_t stream) {
  Ctx* c = pctx(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  if (!p2p_ready(c)) return fail(ROAST_ERR_STATE, "p2p: call roast_p2p_open / roast_p2p_attach after registering every module");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t stride = (c->p2p_n + 3) / 4 * 4;
  PeerWins pw{};
  for (int r = 0; r < c->p2p_world; ++r) pw.w[r] = c->p2p_peer[r];
  const int V = c->touched_vec ? 4 : 1;
  int64_t blocks = (c->p2p_n / V + 255) / 256;
  blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), 148 * 8);
  if (V == 4)
    p2p_post_kernel<4><<<unsigned(blocks), 256, 0, s>>>(c->dM, pw, c->p2p_world, c->p2p_rank, stride, c->d_iv,
                                                        c->d_iv + c->n_iv, c->n_iv, c->p2p_n, mc_int(c, 0));
  else
    p2p_post_kernel<1><<<unsigned(blocks), 256, 0, s>>>(c->dM, pw, c->p2p_world, c->p2p_rank, stride, c->d_iv,
                                                        c->d_iv + c->n_iv, c->n_iv, c->p2p_n, mc_int(c, 0));
  ROAST_CUDA_CHECK(cudaGetLastError());
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_p2p_finish(roast_t h, const roast_opt_config_t* cfg, int64_t step, roast_stream_t stream) {
  Ctx* c = pctx(h);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (roast_status_t st = opt_prepare(c, cfg, step, true, s)) return st;
  if (!p2p_ready(c)) return fail(ROAST_ERR_STATE, "p2p: call roast_p2p_open / roast_p2p_attach after registering every module");
  P2PView v;
  v.world = c->p2p_world;
  for (int r = 0; r < c->p2p_world; ++r) v.buf0[r] = reinterpret_cast<const float*>(c->p2p_peer[r] + kP2PHeader);
  v.stride = (c->p2p_n + 3) / 4 * 4;
  v.flags = reinterpret_cast<const int*>(c->p2p_win);
  v.epoch = reinterpret_cast<const int*>(c->p2p_win + 256);
  v.err = c->d_err;
  if (c->nvls_bound) v.mc_buf0 = reinterpret_cast<const float*>(c->nvls_mc_va + kP2PHeader);   // NVLS one-shot
  if (c->p2p_n == 0) return ROAST_OK;
  ROAST_CUDA_CHECK(launch_optimizer(c, cfg->kind, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay, step,
                                    cfg->zero_grad, true, s, nullptr, &v));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_grad_exchange_p2p(roast_t h, const roast_opt_config_t* cfg, int64_t step,
                                       roast_stream_t stream) {
  Ctx* c = pctx(h);
  if (roast_status_t st = opt_prepare(c, cfg, step, true, reinterpret_cast<cudaStream_t>(stream))) return st;
  if (roast_status_t st = roast_p2p_post(h, stream)) return st;
  return roast_p2p_finish(h, cfg, step, stream);
}

// ---- two-shot: reduce-scatter + update of a slice, then gather (traffic 2 (W - 1) / W n per rank)
namespace {
Slices p2p_slices(const Ctx* c) {
  Slices sl{};
  const int W = c->p2p_world;
  const int64_t n = c->p2p_n;
  const int64_t per = ((n + W - 1) / W + 3) / 4 * 4;
  for (int r = 0; r <= W; ++r) sl.at[r] = std::min<int64_t>(n, int64_t(r) * per);
  for (int r = W + 1; r <= kP2PMaxWorld; ++r) sl.at[r] = n;
  return sl;
}
}  // namespace

roast_status_t roast_p2p_reduce(roast_t h, const roast_opt_config_t* cfg, int64_t step, roast_stream_t stream) {
  Ctx* c = pctx(h);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (roast_status_t st = opt_prepare(c, cfg, step, true, s)) return st;
  if (!p2p_ready(c)) return fail(ROAST_ERR_STATE, "p2p: call roast_p2p_open / roast_p2p_attach after registering every module");
  if (!cfg->zero_grad) return fail(ROAST_ERR_CONFIG, "two-shot p2p exchange: zero_grad must be 1");
  const Slices sl = p2p_slices(c);
  P2PView v;
  v.world = c->p2p_world;
  for (int r = 0; r < c->p2p_world; ++r) v.buf0[r] = reinterpret_cast<const float*>(c->p2p_peer[r] + kP2PHeader);
  v.stride = (c->p2p_n + 3) / 4 * 4;
  v.flags = reinterpret_cast<const int*>(c->p2p_win);
  v.epoch = reinterpret_cast<const int*>(c->p2p_win + 256);
  v.err = c->d_err;
  v.lo = sl.at[c->p2p_rank];
  v.hi = sl.at[c->p2p_rank + 1];
  v.mout = reinterpret_cast<float*>(c->p2p_win + kP2PHeader) + 2 * v.stride;
  if (c->nvls_bound) {   // NVLS: reduce the slice in the switch, broadcast its new values
    v.mc_buf0 = reinterpret_cast<const float*>(c->nvls_mc_va + kP2PHeader);
    v.mc_mout = reinterpret_cast<float*>(c->nvls_mc_va + kP2PHeader) + 2 * v.stride;
  }
  if (c->p2p_n > 0) {   // an empty slice still runs: the kernel waits for every post first
    ROAST_CUDA_CHECK(launch_optimizer(c, cfg->kind, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay,
                                      step, 1, true, s, nullptr, &v));
    c->launches++;
  }
  PeerWins pw{};
  for (int r = 0; r < c->p2p_world; ++r) pw.w[r] = c->p2p_peer[r];
  p2p_signal2_kernel<<<1, 32, 0, s>>>(pw, c->p2p_world, c->p2p_rank, mc_int(c, 128));
  ROAST_CUDA_CHECK(cudaGetLastError());
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_p2p_gather(roast_t h, roast_stream_t stream) {
  Ctx* c = pctx(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  if (!p2p_ready(c)) return fail(ROAST_ERR_STATE, "p2p: call roast_p2p_open / roast_p2p_attach after registering every module");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (c->p2p_n == 0) return ROAST_OK;
  PeerWins pw{};
  for (int r = 0; r < c->p2p_world; ++r) pw.w[r] = c->p2p_peer[r];
  const Slices sl = p2p_slices(c);
  const int64_t stride = (c->p2p_n + 3) / 4 * 4;
  const int V = c->touched_vec ? 4 : 1;
  int64_t blocks = (c->p2p_n / V + 255) / 256;
  blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), 148 * 8);
  if (V == 4)
    p2p_gather_kernel<4><<<unsigned(blocks), 256, 0, s>>>(c->M, c->dM, shadow_out(c), pw, c->p2p_world,
                                                          c->p2p_rank, sl, stride, c->d_iv, c->d_iv + c->n_iv,
                                                          c->n_iv, c->p2p_n, c->d_err);
  else
    p2p_gather_kernel<1><<<unsigned(blocks), 256, 0, s>>>(c->M, c->dM, shadow_out(c), pw, c->p2p_world,
                                                          c->p2p_rank, sl, stride, c->d_iv, c->d_iv + c->n_iv,
                                                          c->n_iv, c->p2p_n, c->d_err);
  ROAST_CUDA_CHECK(cudaGetLastError());
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_grad_exchange_p2p2(roast_t h, const roast_opt_config_t* cfg, int64_t step,
                                        roast_stream_t stream) {
  Ctx* c = pctx(h);
  if (roast_status_t st = opt_prepare(c, cfg, step, true, reinterpret_cast<cudaStream_t>(stream))) return st;
  if (roast_status_t st = roast_p2p_post(h, stream)) return st;
  if (roast_status_t st = roast_p2p_reduce(h, cfg, step, stream)) return st;
  return roast_p2p_gather(h, stream);
}

}  // extern "C"
