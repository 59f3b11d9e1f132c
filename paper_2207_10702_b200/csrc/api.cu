// api.cu — the C ABI of libroast.so (include/roast.h): validation, module
// registration (static tile maps, a0), dispatch to the kernels, sticky errors.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <string>

#include "roast_internal.h"

namespace roast {

static thread_local std::string g_last_error;

roast_status_t fail(roast_status_t st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

roast_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(ROAST_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

roast_status_t scratch_alloc(Scratch& w, size_t bytes, cudaStream_t s) {
  w.s = s;
  // keep freed scratch in the device's default pool (release threshold: unlimited) instead of
  // returning it to the driver at every synchronisation: re-mapping it on the next call cost up to
  // hundreds of us of host time per call (seen as launch gaps in back-to-back LayerNorm backwards)
  static std::atomic<unsigned long long> kept{0};
  if (first_on_device(kept)) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  ROAST_CUDA_CHECK(cudaMallocAsync(&w.p, bytes, s));
  // test hook: fill new scratch with NaN (0xFFFFFFFF) so any slot a reader consumes before a
  // kernel wrote it poisons the result (tests/test_gpu_parity.py, poisoned-workspace test)
  if (getenv("ROAST_POISON_WS")) ROAST_CUDA_CHECK(cudaMemsetAsync(w.p, 0xFF, bytes, s));
  return ROAST_OK;
}

static Ctx* ctx(roast_t h) { return reinterpret_cast<Ctx*>(h); }

static roast_status_t get_module(Ctx* c, int32_t id, ModuleKind kind, Module** out) {
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (id >= kGroupIdBase) {   // roast_register_linear_concat groups (their own id space)
    if (kind != kLinear || id - kGroupIdBase >= int32_t(c->groups.size()))
      return fail(ROAST_ERR_STATE, "unknown linear group id");
    if (!c->M || !c->dM) return fail(ROAST_ERR_STATE, "roast_bind has not been called");
    *out = &c->groups[id - kGroupIdBase];
    return ROAST_OK;
  }
  if (id < 0 || id >= int32_t(c->modules.size())) return fail(ROAST_ERR_STATE, "unknown module id");
  if (c->modules[id].kind != kind) return fail(ROAST_ERR_STATE, "module kind mismatch");
  if (!c->M || !c->dM) return fail(ROAST_ERR_STATE, "roast_bind has not been called");
  *out = &c->modules[id];
  return ROAST_OK;
}

static void free_module(Module& m) {
  cudaFree(m.d_off);
  cudaFree(m.d_sgn);
  cudaFree(m.d_sorted);
  cudaFree(m.d_sorted_off);
  cudaFree(m.d_cover);
  cudaFree(m.d_coord_xy);
  cudaFree(m.d_coord_yx);
}

}  // namespace roast

using namespace roast;

namespace roast {
// validation + lazily allocated optimizer state + (touched) interval tables, shared by
// roast_optimizer_step and roast_grad_exchange_step
roast_status_t opt_prepare(Ctx* c, const roast_opt_config_t* cfg, int64_t step, bool need_touched, cudaStream_t s) {
  if (!c || !c->M || !c->shadow) return fail(ROAST_ERR_STATE, "not bound");
  if (!cfg || cfg->kind < ROAST_OPT_SGD || cfg->kind > ROAST_OPT_ADAM) return fail(ROAST_ERR_CONFIG, "bad optimizer");
  if (cfg->kind == ROAST_OPT_ADAM && step < 1) return fail(ROAST_ERR_CONFIG, "Adam step must be >= 1");
  const size_t bytes = size_t(c->mem_size) * sizeof(float);
  if (cfg->kind >= ROAST_OPT_ADAGRAD && !c->opt_s1) {
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->opt_s1), bytes));
    ROAST_CUDA_CHECK(cudaMemsetAsync(c->opt_s1, 0, bytes, s));
  }
  if (cfg->kind == ROAST_OPT_ADAM && !c->opt_s2) {
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->opt_s2), bytes));
    ROAST_CUDA_CHECK(cudaMemsetAsync(c->opt_s2, 0, bytes, s));
  }
  if (need_touched && !(c->touched_valid && c->touched_for == int64_t(c->modules.size()))) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return fail(ROAST_ERR_STATE, "touched set: call roast_touched_size before capturing");
    if (roast_status_t st = touched_prepare(c, s)) return st;
  }
  return ROAST_OK;
}
}  // namespace roast

namespace roast {
// Device copies of a linear's tile map (h_off / h_sgn [x][y] filled): offsets, signs, the
// offset-sorted order for the deterministic reduce, and the packed TMA coordinates.
roast_status_t upload_linear_tables(Ctx* c, Module& m) {
  const int64_t A = c->cfg.align_elems;
  const int64_t nt = int64_t(m.nx) * m.ny;
  // offset-sorted tile order for the deterministic reduce (ties: tile id)
  std::vector<int32_t> order(nt);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return m.h_off[a] < m.h_off[b]; });
  std::vector<int64_t> soff(nt);
  for (int64_t i = 0; i < nt; ++i) soff[i] = m.h_off[order[i]];
  cudaError_t e = cudaSuccess;
  e = cudaMalloc(reinterpret_cast<void**>(&m.d_off), nt * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&m.d_sgn), nt * sizeof(int8_t));
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&m.d_sorted), nt * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&m.d_sorted_off), nt * sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMemcpy(m.d_off, m.h_off.data(), nt * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m.d_sgn, m.h_sgn.data(), nt * sizeof(int8_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m.d_sorted, order.data(), nt * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(m.d_sorted_off, soff.data(), nt * sizeof(int64_t), cudaMemcpyHostToDevice);
  const int64_t span = int64_t(c->tile.z1) * c->tile.z2, ngroups = (c->mem_size + 3) / 4;
  if (e == cudaSuccess && c->cfg.deterministic && A % 4 == 0 && ngroups * 8 <= (int64_t(64) << 20) &&
      nt * span >= 16 * c->mem_size) {
    // covering range of every 4-slot group (two pointers over the offset-sorted tiles): tiles
    // with off <= s < off + span, i.e. sorted positions [first off > s - span, first off > s)
    std::vector<int32_t> cov(size_t(ngroups) * 2);
    int64_t lo = 0, hi = 0;
    for (int64_t g = 0; g < ngroups; ++g) {
      const int64_t s = 4 * g;
      while (lo < nt && soff[lo] <= s - span) ++lo;
      if (hi < lo) hi = lo;
      while (hi < nt && soff[hi] <= s) ++hi;
      cov[2 * g] = int32_t(lo);
      cov[2 * g + 1] = int32_t(hi);
    }
    e = cudaMalloc(reinterpret_cast<void**>(&m.d_cover), cov.size() * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemcpy(m.d_cover, cov.data(), cov.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && c->mem_size < (int64_t(1) << 33) && A % 8 == 0) {
    std::vector<int32_t> cxy(nt), cyx(nt);
    for (int32_t x = 0; x < m.nx; ++x)
      for (int32_t y = 0; y < m.ny; ++y) {
        const int64_t t = int64_t(x) * m.ny + y;
        const int64_t off = m.h_off[t];
        const int32_t packed = int32_t(((off >> 6) << 4) | (m.h_sgn[t] < 0 ? 8 : 0) | ((off >> 3) & 7));
        cxy[t] = packed;
        cyx[int64_t(y) * m.nx + x] = packed;
      }
    e = cudaMalloc(reinterpret_cast<void**>(&m.d_coord_xy), nt * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&m.d_coord_yx), nt * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemcpy(m.d_coord_xy, cxy.data(), nt * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(m.d_coord_yx, cyx.data(), nt * sizeof(int32_t), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    free_module(m);
    return cuda_fail(e, "register_linear upload");
  }
  return ROAST_OK;
}
}  // namespace roast

extern "C" {

void roast_config_default(roast_config_t* cfg) {
  cfg->C = 1.0;
  cfg->align_elems = 8;
  cfg->tile_layout = ROAST_ROW_MAJOR;
  cfg->mapping = ROAST_MAP_HASH;
  cfg->use_sign = 1;
  cfg->deterministic = 0;
  cfg->simt_bf16 = 0;
}

const char* roast_status_str(roast_status_t st) {
  switch (st) {
    case ROAST_OK: return "ok";
    case ROAST_ERR_CONFIG: return "config error";
    case ROAST_ERR_GEOMETRY: return "geometry error";
    case ROAST_ERR_SHAPE: return "shape error";
    case ROAST_ERR_BOUNDS: return "bounds error";
    case ROAST_ERR_CAPACITY: return "capacity error";
    case ROAST_ERR_STATE: return "state error";
    case ROAST_ERR_CUDA: return "CUDA error";
    case ROAST_ERR_NCCL: return "NCCL error";
    case ROAST_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* roast_last_error(void) { return g_last_error.c_str(); }

roast_status_t roast_create_ex(roast_t* out, int64_t mem_size, uint64_t seed, roast_tile_t tile,
                               const roast_config_t* cfg_in) {
  if (!out) return fail(ROAST_ERR_CONFIG, "null out");
  roast_config_t cfg;
  if (cfg_in)
    cfg = *cfg_in;
  else
    roast_config_default(&cfg);
  if (mem_size <= 0) return fail(ROAST_ERR_CONFIG, "mem_size must be > 0");
  if (!(cfg.C > 0)) return fail(ROAST_ERR_CONFIG, "C must be > 0");
  // A = 1 is legal (HashedNet-style 1x1 tiles on the SIMT path); embeddings need A % 4 == 0
  // and the tcgen05 path A % 8 == 0 (16-byte TMA offsets); both are checked where they apply.
  if (cfg.align_elems <= 0) return fail(ROAST_ERR_CONFIG, "align_elems must be positive");
  if (cfg.tile_layout != ROAST_ROW_MAJOR && cfg.tile_layout != ROAST_SW128)
    return fail(ROAST_ERR_CONFIG, "bad tile_layout");
  if (cfg.mapping != ROAST_MAP_HASH && cfg.mapping != ROAST_MAP_IDENTITY) return fail(ROAST_ERR_CONFIG, "bad mapping");
  if (tile.z1 <= 0 || tile.z2 <= 0) return fail(ROAST_ERR_GEOMETRY, "tile dims must be > 0");
  if (cfg.tile_layout == ROAST_SW128 && tile.z2 != 64)
    return fail(ROAST_ERR_GEOMETRY, "SW128 tile layout needs Z2 = 64 (128-byte bf16 rows)");
  Ctx* c = new Ctx();
  c->mem_size = mem_size;
  c->seed = seed;
  c->tile = tile;
  c->cfg = cfg;
  // one 16-byte block: the sticky error flag, then an int64 0 (row 0 of a bias via L)
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&c->d_err), 16);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(err flag)");
  }
  cudaMemset(c->d_err, 0, 16);
  {   // per-call scratch comes from the default pool: keep up to 1 GiB of freed blocks cached
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = uint64_t(1) << 30, cur = 0;
      if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur) == cudaSuccess && cur < keep)
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  c->d_zero_idx = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(c->d_err) + 8);
  *out = reinterpret_cast<roast_t>(c);
  return ROAST_OK;
}

roast_status_t roast_create(roast_t* out, int64_t mem_size, uint64_t seed, roast_tile_t tile) {
  return roast_create_ex(out, mem_size, seed, tile, nullptr);
}

roast_status_t roast_destroy(roast_t h) {
  Ctx* c = ctx(h);
  if (!c) return ROAST_OK;
  cudaDeviceSynchronize();
  for (auto& m : c->modules) free_module(m);
  for (auto& m : c->groups) free_module(m);
  cudaFree(c->shadow);
  cudaFree(c->dm_rep);
  cudaFree(c->d_err);
  cudaFree(c->opt_s1);
  cudaFree(c->opt_s2);
  for (auto& kv : c->chain_plans) cudaFree(kv.second.first);
  cudaFree(c->chain_flags);
  cudaFree(c->d_iv);
  cudaFree(c->d_pack);
  comm_destroy(c);
  p2p_destroy(c);
  delete c;
  return ROAST_OK;
}

// Replicas of the bf16 shadow.  At high compression the whole shadow is a few L2 lines' worth
// (C2 at 1000x: 19 KB) and every CTA pair's hashed-tile loads land on the same L2 slices; R
// copies (CTA pair p reads copy p % R) spread them.  Bounded to 1 MB in total; ROAST_SHADOW_REPS
// overrides (A/B).
static int shadow_replicas(int64_t elems) {
  if (const char* e = getenv("ROAST_SHADOW_REPS")) return std::max(1, std::min(74, atoi(e)));
  const int64_t bytes = elems * int64_t(sizeof(uint16_t));
  int r = 1;
  while (r < 16 && bytes * 2 * r <= (int64_t(1) << 20)) r *= 2;
  return r;
}

roast_status_t roast_bind(roast_t h, float* d_M, float* d_dM, roast_stream_t stream) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (!d_M || !d_dM) return fail(ROAST_ERR_CONFIG, "null M / dM");
  if ((reinterpret_cast<uintptr_t>(d_M) | reinterpret_cast<uintptr_t>(d_dM)) & 15)
    return fail(ROAST_ERR_CONFIG, "M and dM must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  c->M = d_M;
  c->dM = d_dM;
  if (!c->shadow) {
    // [+bf16(M) | pad | -bf16(M) | 64-element tail pad]; the negated copy starts 128-B aligned
    c->neg_base = (c->mem_size + 63) / 64 * 64;
    c->shadow_elems = 2 * c->neg_base + 64;
    c->shadow_reps = shadow_replicas(c->shadow_elems);
    const size_t bytes = size_t(c->shadow_reps) * c->shadow_elems * sizeof(uint16_t);
    ROAST_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&c->shadow), bytes));
    ROAST_CUDA_CHECK(cudaMemsetAsync(c->shadow, 0, bytes, s));
    c->tmap_shadow_valid = false;
  }
  ROAST_CUDA_CHECK(launch_sync_shadow(c, s));
  c->launches++;
  return ROAST_OK;
}

// [seg_base, seg_base + seg_size) must be an A-aligned piece of M holding at least one span
static roast_status_t check_segment(const Ctx* c, int64_t seg_base, int64_t seg_size, int64_t span) {
  const int64_t A = c->cfg.align_elems;
  if (seg_base < 0 || seg_size <= 0 || seg_base > c->mem_size - seg_size)
    return fail(ROAST_ERR_GEOMETRY, "segment outside M");
  if (seg_base % A) return fail(ROAST_ERR_GEOMETRY, "segment base must be a multiple of align_elems");
  if (span > seg_size) return fail(ROAST_ERR_GEOMETRY, "tile / chunk larger than the module's memory (S:51)");
  return ROAST_OK;
}

roast_status_t roast_register_linear(roast_t h, int64_t H, int64_t O, int32_t* id) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  return roast_register_linear_seg(h, H, O, 0, c->mem_size, id);
}

roast_status_t roast_register_linear_seg(roast_t h, int64_t H, int64_t O, int64_t seg_base, int64_t seg_size,
                                         int32_t* id) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (H <= 0 || O <= 0) return fail(ROAST_ERR_SHAPE, "in/out features must be > 0");
  const int64_t z1 = c->tile.z1, z2 = c->tile.z2, T = z1 * z2, A = c->cfg.align_elems;
  if (T > c->mem_size) return fail(ROAST_ERR_GEOMETRY, "tile Z1*Z2 larger than |M| (S:51)");
  if (roast_status_t st = check_segment(c, seg_base, seg_size, T)) return st;
  if (c->cfg.mapping == ROAST_MAP_IDENTITY && (seg_base != 0 || seg_size != c->mem_size))
    return fail(ROAST_ERR_CONFIG, "segments apply to the hashed mapping only");
  if (H % z1 || O % z2) return fail(ROAST_ERR_GEOMETRY, "in % Z1 and out % Z2 must be 0 on the GPU path (R9)");
  if (T % A) return fail(ROAST_ERR_GEOMETRY, "Z1*Z2 must be a multiple of align_elems");
  if (c->cfg.deterministic && A % 4)
    return fail(ROAST_ERR_GEOMETRY, "deterministic dM needs align_elems % 4 == 0 (4-slot reduce groups)");
  if (H / z1 >= (int64_t(1) << 28) || O / z2 >= (int64_t(1) << 31)) return fail(ROAST_ERR_GEOMETRY, "too many tiles");
  Module m;
  m.kind = kLinear;
  m.H = H;
  m.O = O;
  m.nx = int32_t(H / z1);
  m.ny = int32_t(O / z2);
  const uint32_t mid = uint32_t(c->modules.size());
  m.hash.off = make_coef(c->seed, mid, 0);
  m.hash.sgn = make_coef(c->seed, mid, 1);
  m.hash.set_range(uint64_t((seg_size - T) / A + 1));
  m.hash.base = uint64_t(seg_base);
  m.hash.align = uint32_t(A);
  m.hash.use_sign = c->cfg.use_sign ? 1u : 0u;
  const int64_t nt = int64_t(m.nx) * m.ny;
  m.h_off.resize(nt);
  m.h_sgn.resize(nt);
  if (c->cfg.mapping == ROAST_MAP_IDENTITY) {
    if (c->identity_cursor + nt * T > c->mem_size) return fail(ROAST_ERR_GEOMETRY, "identity mapping needs |M| >= n");
    for (int64_t t = 0; t < nt; ++t) {
      m.h_off[t] = c->identity_cursor + T * t;
      m.h_sgn[t] = 1;
    }
    c->identity_cursor += nt * T;
    m.lam = 1.0f;
  } else {
    for (int32_t x = 0; x < m.nx; ++x)
      for (int32_t y = 0; y < m.ny; ++y) {
        uint64_t k = tile_key(uint32_t(x), uint32_t(y));
        m.h_off[int64_t(x) * m.ny + y] = int64_t(m.hash.offset(k));
        m.h_sgn[int64_t(x) * m.ny + y] = int8_t(m.hash.sign(k));
      }
    m.lam = float(c->cfg.C / sqrt(double(H)));
  }
  if (roast_status_t st = upload_linear_tables(c, m)) return st;
  c->modules.push_back(std::move(m));
  if (id) *id = int32_t(mid);
  return ROAST_OK;
}


roast_status_t roast_register_linear_concat(roast_t h, const int32_t* ids, int32_t n, int32_t* group_id) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (!ids || n < 1) return fail(ROAST_ERR_CONFIG, "null / empty member list");
  std::vector<const Module*> mem(n);
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= int32_t(c->modules.size()) || c->modules[ids[i]].kind != kLinear)
      return fail(ROAST_ERR_STATE, "member is not a registered linear");
    mem[i] = &c->modules[ids[i]];
    if (mem[i]->H != mem[0]->H || mem[i]->lam != mem[0]->lam)
      return fail(ROAST_ERR_SHAPE, "members need equal in_features (and lambda)");
  }
  Module g;
  g.kind = kLinear;
  g.lam = mem[0]->lam;
  g.hash = mem[0]->hash;   // unused: the group's tiles come from its members' maps
  g.H = mem[0]->H;
  g.nx = mem[0]->nx;
  for (const Module* m : mem) {
    g.O += m->O;
    g.ny += m->ny;
  }
  const int64_t nt = int64_t(g.nx) * g.ny;
  g.h_off.resize(nt);
  g.h_sgn.resize(nt);
  for (int32_t x = 0; x < g.nx; ++x) {
    int32_t y0 = 0;
    for (const Module* m : mem) {   // row x of the group = row x of every member, side by side
      for (int32_t y = 0; y < m->ny; ++y) {
        g.h_off[int64_t(x) * g.ny + y0 + y] = m->h_off[int64_t(x) * m->ny + y];
        g.h_sgn[int64_t(x) * g.ny + y0 + y] = m->h_sgn[int64_t(x) * m->ny + y];
      }
      y0 += m->ny;
    }
  }
  if (roast_status_t st = upload_linear_tables(c, g)) return st;
  c->groups.push_back(std::move(g));
  if (group_id) *group_id = kGroupIdBase + int32_t(c->groups.size()) - 1;
  return ROAST_OK;
}

roast_status_t roast_register_embedding(roast_t h, int64_t num_rows, int32_t dim, int32_t chunk, double fan_in,
                                        int32_t* id) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  return roast_register_embedding_seg(h, num_rows, dim, chunk, fan_in, 0, c->mem_size, id);
}

roast_status_t roast_register_embedding_seg(roast_t h, int64_t num_rows, int32_t dim, int32_t chunk, double fan_in,
                                            int64_t seg_base, int64_t seg_size, int32_t* id) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (num_rows <= 0 || dim <= 0 || chunk <= 0) return fail(ROAST_ERR_SHAPE, "rows, dim, chunk must be > 0");
  const int64_t A = c->cfg.align_elems;
  if (chunk > c->mem_size) return fail(ROAST_ERR_GEOMETRY, "chunk larger than |M|");
  if (roast_status_t st = check_segment(c, seg_base, seg_size, chunk)) return st;
  if (chunk % A || chunk % 4 || dim % 4 || A % 4)
    return fail(ROAST_ERR_GEOMETRY, "chunk % A, chunk % 4, dim % 4 and A % 4 must be 0 (16-byte vector access)");
  Module m;
  m.kind = kEmbedding;
  m.rows = num_rows;
  m.dim = dim;
  m.chunk = chunk;
  m.chunks_per_row = (dim + chunk - 1) / chunk;
  if (double(num_rows) * m.chunks_per_row >= double(int64_t(1) << 60)) return fail(ROAST_ERR_GEOMETRY, "too many chunks");
  const uint32_t mid = uint32_t(c->modules.size());
  m.hash.off = make_coef(c->seed, mid, 0);
  m.hash.sgn = make_coef(c->seed, mid, 1);
  m.hash.set_range(uint64_t((seg_size - chunk) / A + 1));
  m.hash.base = uint64_t(seg_base);
  m.hash.align = uint32_t(A);
  m.hash.use_sign = c->cfg.use_sign ? 1u : 0u;
  m.lam = float(c->cfg.C / sqrt(fan_in > 0 ? fan_in : double(dim)));
  c->modules.push_back(std::move(m));
  if (id) *id = int32_t(mid);
  return ROAST_OK;
}

static bool use_sm100(const Ctx* c, const Module& m) {
  return c->tile.z1 == 64 && c->tile.z2 == 64 && m.H % 64 == 0 && m.O % 64 == 0 &&
         getenv("ROAST_FORCE_SIMT") == nullptr;
}

// A bf16 call the tcgen05 path did not take runs on the SIMT kernels only if the handle opted in
// (roast_config_t.simt_bf16, or the ROAST_FORCE_SIMT diagnostic); otherwise it is an error, not
// a silent second backend.  fp32 calls always use the SIMT kernels (the fp32 path).
static roast_status_t simt_allowed(const Ctx* c, roast_dtype_t dt) {
  if (dt != ROAST_BF16 || c->cfg.simt_bf16 || getenv("ROAST_FORCE_SIMT")) return ROAST_OK;
  return fail(ROAST_ERR_UNSUPPORTED,
              "bf16 linear off the tcgen05 path (needs 64x64 row-major tiles, A % 8 == 0, tokens < 2^31); "
              "set roast_config_t.simt_bf16 = 1 to run it on the SIMT kernels");
}

roast_status_t roast_linear_fwd(roast_t h, int32_t id, const void* X, void* Y, int64_t T, roast_dtype_t dt,
                                roast_stream_t stream) {
  return roast_linear_fwd_bias(h, id, X, Y, T, dt, nullptr, stream);
}

roast_status_t roast_linear_fwd_bias(roast_t h, int32_t id, const void* X, void* Y, int64_t T, roast_dtype_t dt,
                                     const float* bias, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, id, kLinear, &m);
  if (st) return st;
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (T > 0 && (!X || !Y)) return fail(ROAST_ERR_CONFIG, "null X / Y");
  if (dt != ROAST_FP32 && dt != ROAST_BF16) return fail(ROAST_ERR_CONFIG, "bad dtype");
  if (reinterpret_cast<uintptr_t>(bias) & 15) return fail(ROAST_ERR_CONFIG, "bias must be 16-byte aligned");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (T == 0) return ROAST_OK;
  if (dt == ROAST_BF16 && use_sm100(c, *m)) {
    st = sm100_fwd(c, *m, X, Y, T, bias, s);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = simt_allowed(c, dt))) return st;
  ROAST_CUDA_CHECK(launch_simt_fwd(c, *m, X, Y, T, dt, false, s, bias));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_linear_fwd_act(roast_t h, int32_t id, const void* X, void* Y, void* A, int64_t T,
                                    roast_dtype_t dt, const float* bias, int32_t act, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, id, kLinear, &m);
  if (st) return st;
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (act != ROAST_ACT_GELU_TANH) return fail(ROAST_ERR_CONFIG, "act: ROAST_ACT_GELU_TANH");
  if (T > 0 && (!X || !Y || !A)) return fail(ROAST_ERR_CONFIG, "null X / Y / A");
  if ((reinterpret_cast<uintptr_t>(bias) | reinterpret_cast<uintptr_t>(A)) & 15)
    return fail(ROAST_ERR_CONFIG, "bias and A must be 16-byte aligned");
  if (T == 0) return ROAST_OK;
  if (dt != ROAST_BF16 || !use_sm100(c, *m))
    return fail(ROAST_ERR_UNSUPPORTED, "fused activation: bf16 on the tcgen05 path only");
  st = sm100_fwd_act(c, *m, X, Y, A, T, bias, act, reinterpret_cast<cudaStream_t>(stream));
  if (st == ROAST_ERR_UNSUPPORTED) return fail(st, "fused activation: not on this geometry");
  return st;
}

roast_status_t roast_linear_fwd_chain(roast_t h, int32_t id_a, int32_t id_b, const void* X, void* Y_a, void* Y_b,
                                      int64_t T, roast_dtype_t dt, const float* bias_a, const float* bias_b,
                                      roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module *ma, *mb;
  roast_status_t st = get_module(c, id_a, kLinear, &ma);
  if (st) return st;
  if ((st = get_module(c, id_b, kLinear, &mb))) return st;
  if (ma->O != mb->H) return fail(ROAST_ERR_SHAPE, "chain: out_features of a != in_features of b");
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (T > 0 && (!X || !Y_a || !Y_b)) return fail(ROAST_ERR_CONFIG, "null X / Y_a / Y_b");
  if ((reinterpret_cast<uintptr_t>(bias_a) | reinterpret_cast<uintptr_t>(bias_b)) & 15)
    return fail(ROAST_ERR_CONFIG, "bias must be 16-byte aligned");
  if (T == 0) return ROAST_OK;
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dt == ROAST_BF16 && use_sm100(c, *ma) && use_sm100(c, *mb)) {
    st = sm100_chain(c, *ma, *mb, X, Y_a, Y_b, T, false, bias_a, bias_b, s);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = roast_linear_fwd_bias(h, id_a, X, Y_a, T, dt, bias_a, stream))) return st;
  return roast_linear_fwd_bias(h, id_b, Y_a, Y_b, T, dt, bias_b, stream);
}

roast_status_t roast_linear_bwd_dx_chain(roast_t h, int32_t id_a, int32_t id_b, const void* dY_b, void* dY_a,
                                         void* dX, int64_t T, roast_dtype_t dt, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module *ma, *mb;
  roast_status_t st = get_module(c, id_a, kLinear, &ma);
  if (st) return st;
  if ((st = get_module(c, id_b, kLinear, &mb))) return st;
  if (ma->O != mb->H) return fail(ROAST_ERR_SHAPE, "chain: out_features of a != in_features of b");
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (T > 0 && (!dY_b || !dY_a || !dX)) return fail(ROAST_ERR_CONFIG, "null dY_b / dY_a / dX");
  if (T == 0) return ROAST_OK;
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dt == ROAST_BF16 && use_sm100(c, *ma) && use_sm100(c, *mb)) {
    st = sm100_chain(c, *mb, *ma, dY_b, dY_a, dX, T, true, nullptr, nullptr, s);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = roast_linear_bwd_dx(h, id_b, dY_b, dY_a, T, dt, stream))) return st;
  return roast_linear_bwd_dx(h, id_a, dY_a, dX, T, dt, stream);
}

roast_status_t roast_linear_bwd_chain(roast_t h, int32_t id_a, int32_t id_b, const void* X_a, const void* Y_a,
                                      const void* dY_b, void* dY_a, void* dX_a, int64_t T, roast_dtype_t dt,
                                      roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module *ma, *mb;
  roast_status_t st = get_module(c, id_a, kLinear, &ma);
  if (st) return st;
  if ((st = get_module(c, id_b, kLinear, &mb))) return st;
  if (ma->O != mb->H) return fail(ROAST_ERR_SHAPE, "chain: out_features of a != in_features of b");
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (T > 0 && (!X_a || !Y_a || !dY_b || !dY_a || !dX_a)) return fail(ROAST_ERR_CONFIG, "null tensor argument");
  if (dt != ROAST_FP32 && dt != ROAST_BF16) return fail(ROAST_ERR_CONFIG, "bad dtype");
  if (T == 0) return ROAST_OK;
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dt == ROAST_BF16 && use_sm100(c, *ma) && use_sm100(c, *mb)) {
    st = sm100_bwd_chain(c, *ma, *mb, X_a, Y_a, dY_b, dY_a, dX_a, T, s);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = roast_linear_bwd_dx(h, id_b, dY_b, dY_a, T, dt, stream))) return st;
  if ((st = roast_linear_bwd_dm(h, id_b, Y_a, dY_b, T, dt, stream))) return st;
  if ((st = roast_linear_bwd_dx(h, id_a, dY_a, dX_a, T, dt, stream))) return st;
  return roast_linear_bwd_dm(h, id_a, X_a, dY_a, T, dt, stream);
}

roast_status_t roast_linear_fwd_chain_act(roast_t h, int32_t id_a, int32_t id_b, const void* X, void* U, void* A,
                                          void* Y_b, int64_t T, roast_dtype_t dt, const float* bias_a,
                                          const float* bias_b, int32_t act, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module *ma, *mb;
  roast_status_t st = get_module(c, id_a, kLinear, &ma);
  if (st) return st;
  if ((st = get_module(c, id_b, kLinear, &mb))) return st;
  if (ma->O != mb->H) return fail(ROAST_ERR_SHAPE, "chain: out_features of a != in_features of b");
  if (act != ROAST_ACT_GELU_TANH) return fail(ROAST_ERR_CONFIG, "act: ROAST_ACT_GELU_TANH");
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (T > 0 && (!X || !U || !A || !Y_b)) return fail(ROAST_ERR_CONFIG, "null X / U / A / Y_b");
  if ((reinterpret_cast<uintptr_t>(bias_a) | reinterpret_cast<uintptr_t>(bias_b)) & 15)
    return fail(ROAST_ERR_CONFIG, "bias must be 16-byte aligned");
  if (T == 0) return ROAST_OK;
  if (dt == ROAST_BF16 && use_sm100(c, *ma) && use_sm100(c, *mb)) {
    st = sm100_chain(c, *ma, *mb, X, U, Y_b, T, false, bias_a, bias_b, reinterpret_cast<cudaStream_t>(stream), act, A);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = roast_linear_fwd_act(h, id_a, X, U, A, T, dt, bias_a, act, stream))) return st;
  return roast_linear_fwd_bias(h, id_b, A, Y_b, T, dt, bias_b, stream);
}

roast_status_t roast_linear_bwd_chain_act(roast_t h, int32_t id_a, int32_t id_b, const void* X_a, const void* A,
                                          const void* U, const void* dY_b, void* dU, void* dX_a, int64_t T,
                                          roast_dtype_t dt, int32_t act, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module *ma, *mb;
  roast_status_t st = get_module(c, id_a, kLinear, &ma);
  if (st) return st;
  if ((st = get_module(c, id_b, kLinear, &mb))) return st;
  if (ma->O != mb->H) return fail(ROAST_ERR_SHAPE, "chain: out_features of a != in_features of b");
  if (act != ROAST_ACT_GELU_TANH) return fail(ROAST_ERR_CONFIG, "act: ROAST_ACT_GELU_TANH");
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (T > 0 && (!X_a || !A || !U || !dY_b || !dU || !dX_a)) return fail(ROAST_ERR_CONFIG, "null tensor argument");
  if (T == 0) return ROAST_OK;
  if (dt == ROAST_BF16 && use_sm100(c, *ma) && use_sm100(c, *mb)) {
    st = sm100_bwd_chain(c, *ma, *mb, X_a, A, dY_b, dU, dX_a, T, reinterpret_cast<cudaStream_t>(stream), act, U);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = roast_linear_bwd_dx_act(h, id_b, dY_b, U, dU, T, dt, act, stream))) return st;
  if ((st = roast_linear_bwd_dm(h, id_b, A, dY_b, T, dt, stream))) return st;
  if ((st = roast_linear_bwd_dx(h, id_a, dU, dX_a, T, dt, stream))) return st;
  return roast_linear_bwd_dm(h, id_a, X_a, dU, T, dt, stream);
}

roast_status_t roast_bias_fwd(roast_t h, int32_t bias_id, float* b, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, bias_id, kEmbedding, &m);
  if (st) return st;
  if (!b) return fail(ROAST_ERR_CONFIG, "null bias output");
  if (reinterpret_cast<uintptr_t>(b) & 15) return fail(ROAST_ERR_CONFIG, "bias must be 16-byte aligned");
  ROAST_CUDA_CHECK(launch_embed_fwd(c, *m, c->d_zero_idx, 1, b, reinterpret_cast<cudaStream_t>(stream)));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_bias_bwd(roast_t h, int32_t bias_id, const void* dY, int64_t T, roast_dtype_t dt,
                              roast_stream_t stream) {
  return roast_bias_bwd_ld(h, bias_id, dY, T, -1, dt, stream);
}

roast_status_t roast_colsum(const void* dY, int64_t T, int32_t n, int64_t ld, roast_dtype_t dt, float* db,
                            roast_stream_t stream) {
  return roast_colsum_ex(dY, T, n, ld, dt, db, 0, stream);
}

roast_status_t roast_colsum_ex(const void* dY, int64_t T, int32_t n, int64_t ld, roast_dtype_t dt, float* db,
                               int32_t accumulate, roast_stream_t stream) {
  if (T < 0 || n <= 0) return fail(ROAST_ERR_SHAPE, "tokens < 0 or n <= 0");
  if (dt != ROAST_FP32 && dt != ROAST_BF16) return fail(ROAST_ERR_CONFIG, "bad dtype");
  if (ld < 0) ld = n;
  if (ld < n || (ld % 2) || (n % 2)) return fail(ROAST_ERR_SHAPE, "ld must be >= n; n and ld even");
  if (!db || (reinterpret_cast<uintptr_t>(db) & 7)) return fail(ROAST_ERR_CONFIG, "db must be 8-byte aligned");
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (T == 0) {
    if (!accumulate) ROAST_CUDA_CHECK(cudaMemsetAsync(db, 0, size_t(n) * sizeof(float), s));
    return ROAST_OK;
  }
  if (!dY || (reinterpret_cast<uintptr_t>(dY) & 7)) return fail(ROAST_ERR_CONFIG, "dY must be 8-byte aligned");
  const int slabs = colsum_slabs(T, n);
  float* tmp = nullptr;   // stream-ordered scratch for the slab partials (capturable)
  ROAST_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), size_t(slabs) * n * sizeof(float), s));
  cudaError_t e = launch_colsum(dY, T, n, ld, dt, tmp, db, s, accumulate ? 1 : 0);
  cudaFreeAsync(tmp, s);
  if (e != cudaSuccess) return cuda_fail(e, "column sum");
  return ROAST_OK;
}

roast_status_t roast_bias_bwd_ld(roast_t h, int32_t bias_id, const void* dY, int64_t T, int64_t ld, roast_dtype_t dt,
                                 roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, bias_id, kEmbedding, &m);
  if (st) return st;
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (dt != ROAST_FP32 && dt != ROAST_BF16) return fail(ROAST_ERR_CONFIG, "bad dtype");
  if (T == 0) return ROAST_OK;
  if (!dY) return fail(ROAST_ERR_CONFIG, "null dY");
  if (reinterpret_cast<uintptr_t>(dY) & 7) return fail(ROAST_ERR_CONFIG, "dY must be 8-byte aligned");
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int n = m->dim;
  if (ld < 0) ld = n;
  if (ld < n || (ld % 2)) return fail(ROAST_ERR_SHAPE, "ld must be >= the bias length and even");
  const int slabs = colsum_slabs(T, n);
  float* tmp = nullptr;   // stream-ordered scratch: slab partials, then db (capturable)
  ROAST_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), (size_t(slabs) + 1) * n * sizeof(float) + 16, s));
  float* db = tmp + size_t(slabs) * n;
  db = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(db) + 15) & ~uintptr_t(15));
  cudaError_t e = launch_colsum(dY, T, n, ld, dt, tmp, db, s);
  c->launches += 2;
  if (e == cudaSuccess) {
    if (c->cfg.deterministic) {
      {
        const Module* one = m;
        st = embed_bwd_deterministic(c, &one, 1, c->d_zero_idx, 1, db, s);
      }
    } else {
      e = launch_embed_bwd(c, *m, c->d_zero_idx, 1, db, s);
      c->launches++;
    }
  }
  cudaFreeAsync(tmp, s);
  if (e != cudaSuccess) return cuda_fail(e, "bias backward");
  return st;
}

static roast_status_t linear_args(Ctx* c, int32_t id, int64_t T, roast_dtype_t dt, const void* a, const void* b,
                                  Module** m) {
  roast_status_t st = get_module(c, id, kLinear, m);
  if (st) return st;
  if (T < 0) return fail(ROAST_ERR_SHAPE, "tokens < 0");
  if (T > 0 && (!a || !b)) return fail(ROAST_ERR_CONFIG, "null tensor argument");
  if (dt != ROAST_FP32 && dt != ROAST_BF16) return fail(ROAST_ERR_CONFIG, "bad dtype");
  return ROAST_OK;
}

roast_status_t roast_linear_bwd_dx(roast_t h, int32_t id, const void* dY, void* dX, int64_t T, roast_dtype_t dt,
                                   roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = linear_args(c, id, T, dt, dY, dX, &m);
  if (st || T == 0) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // a2: dX = lambda dY W~^T
  if (dt == ROAST_BF16 && use_sm100(c, *m)) {
    st = sm100_dx(c, *m, dY, dX, T, s);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = simt_allowed(c, dt))) return st;
  ROAST_CUDA_CHECK(launch_simt_fwd(c, *m, dY, dX, T, dt, true, s, nullptr));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_linear_bwd_dx_act(roast_t h, int32_t id, const void* dY, const void* U, void* dX, int64_t T,
                                       roast_dtype_t dt, int32_t act, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = linear_args(c, id, T, dt, dY, dX, &m);
  if (st || T == 0) return st;
  if (act != ROAST_ACT_GELU_TANH && act != ROAST_ACT_RESIDUAL)
    return fail(ROAST_ERR_CONFIG, "act: ROAST_ACT_GELU_TANH or ROAST_ACT_RESIDUAL");
  if (!U || (reinterpret_cast<uintptr_t>(U) & 15)) return fail(ROAST_ERR_CONFIG, "U null or not 16-byte aligned");
  if (dt != ROAST_BF16 || !use_sm100(c, *m))
    return fail(ROAST_ERR_UNSUPPORTED, "fused activation: bf16 on the tcgen05 path only");
  st = sm100_dx_act(c, *m, dY, U, dX, T, act, reinterpret_cast<cudaStream_t>(stream));
  if (st == ROAST_ERR_UNSUPPORTED) return fail(st, "fused activation: not on this geometry");
  return st;
}

roast_status_t roast_linear_bwd_dm(roast_t h, int32_t id, const void* X, const void* dY, int64_t T, roast_dtype_t dt,
                                   roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = linear_args(c, id, T, dt, X, dY, &m);
  if (st || T == 0) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // a3: dM += scatter(lambda g X^T dY)
  if (dt == ROAST_BF16 && use_sm100(c, *m)) {
    st = sm100_dw(c, *m, X, dY, T, s);
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  if ((st = simt_allowed(c, dt))) return st;
  if (c->cfg.deterministic) {
    const size_t bytes = size_t(m->nx) * m->ny * c->tile.z1 * c->tile.z2 * sizeof(float);
    Scratch ws;
    if ((st = scratch_alloc(ws, bytes, s))) return st;
    ROAST_CUDA_CHECK(launch_simt_dw(c, *m, X, dY, T, dt, ws.as<float>(), s));
    ROAST_CUDA_CHECK(launch_det_reduce(c, *m, ws.as<float>(), 1, s));
    c->launches += 2;
  } else {
    ROAST_CUDA_CHECK(launch_simt_dw(c, *m, X, dY, T, dt, nullptr, s));
    c->launches++;
  }
  return ROAST_OK;
}

roast_status_t roast_linear_bwd_fused(roast_t h, int32_t id, const void* X, const void* dY, void* dX, int64_t T,
                                      roast_dtype_t dt, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = linear_args(c, id, T, dt, X, dY, &m);
  if (st || T == 0) return st;
  if (!dX) return fail(ROAST_ERR_CONFIG, "bwd_fused: dX is required");
  if (dt == ROAST_BF16 && use_sm100(c, *m)) {
    st = sm100_bwd_fused1(c, *m, X, dY, dX, T, reinterpret_cast<cudaStream_t>(stream));
    if (st != ROAST_ERR_UNSUPPORTED) return st;
  }
  return roast_linear_bwd(h, id, X, dY, dX, T, dt, stream);   // the two launches
}

roast_status_t roast_linear_bwd(roast_t h, int32_t id, const void* X, const void* dY, void* dX, int64_t T,
                                roast_dtype_t dt, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = linear_args(c, id, T, dt, X, dY, &m);
  if (st || T == 0) return st;
  if (dX) {
    st = roast_linear_bwd_dx(h, id, dY, dX, T, dt, stream);
    if (st) return st;
  }
  return roast_linear_bwd_dm(h, id, X, dY, T, dt, stream);
}

roast_status_t roast_embedding_fwd(roast_t h, int32_t id, const int64_t* idx, int64_t n, float* out,
                                   roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, id, kEmbedding, &m);
  if (st) return st;
  if (n < 0) return fail(ROAST_ERR_SHAPE, "n < 0");
  if (n > 0 && (!idx || !out)) return fail(ROAST_ERR_CONFIG, "null idx / out");
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(ROAST_ERR_CONFIG, "out must be 16-byte aligned");
  ROAST_CUDA_CHECK(launch_embed_fwd(c, *m, idx, n, out, reinterpret_cast<cudaStream_t>(stream)));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_embedding_bwd(roast_t h, int32_t id, const int64_t* idx, int64_t n, const float* dOut,
                                   roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, id, kEmbedding, &m);
  if (st) return st;
  if (n < 0) return fail(ROAST_ERR_SHAPE, "n < 0");
  if (n > 0 && (!idx || !dOut)) return fail(ROAST_ERR_CONFIG, "null idx / dOut");
  if (reinterpret_cast<uintptr_t>(dOut) & 15) return fail(ROAST_ERR_CONFIG, "dOut must be 16-byte aligned");
  if (c->cfg.deterministic) {
    const Module* one = m;
    return embed_bwd_deterministic(c, &one, 1, idx, n, dOut, reinterpret_cast<cudaStream_t>(stream));
  }
  ROAST_CUDA_CHECK(launch_embed_bwd(c, *m, idx, n, dOut, reinterpret_cast<cudaStream_t>(stream)));
  c->launches++;
  return ROAST_OK;
}

static roast_status_t embedding_multi(roast_t h, const int32_t* ids, int32_t nt, const int64_t* idx, int64_t n,
                                      float* out, const float* dOut, roast_stream_t stream) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (nt < 0 || n < 0) return fail(ROAST_ERR_SHAPE, "ntables < 0 or n < 0");
  if (nt == 0 || n == 0) return ROAST_OK;
  if (!ids || !idx || (!out && !dOut)) return fail(ROAST_ERR_CONFIG, "null ids / idx / out");
  const void* rows = out ? static_cast<const void*>(out) : static_cast<const void*>(dOut);
  if (reinterpret_cast<uintptr_t>(rows) & 15) return fail(ROAST_ERR_CONFIG, "out / dOut must be 16-byte aligned");
  std::vector<const Module*> mods(nt);
  for (int t = 0; t < nt; ++t) {
    Module* m;
    roast_status_t st = get_module(c, ids[t], kEmbedding, &m);
    if (st) return st;
    if (t && (m->dim != mods[0]->dim || m->chunk != mods[0]->chunk))
      return fail(ROAST_ERR_CONFIG, "multi-table call needs equal dim and chunk");
    mods[t] = m;
  }
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t dim = mods[0]->dim;
  if (dOut && c->cfg.deterministic)  // fixed order: the tables' items sorted together (K7 det)
    return embed_bwd_deterministic(c, mods.data(), nt, idx, n, dOut, s);
  for (int t0 = 0; t0 < nt; t0 += kEmbMaxTables) {
    const int k = std::min(nt - t0, kEmbMaxTables);
    ROAST_CUDA_CHECK(launch_embed_multi(c, mods.data() + t0, k, idx + t0 * n, n, out ? out + t0 * n * dim : nullptr,
                                        dOut ? dOut + t0 * n * dim : nullptr, s));
    c->launches++;
  }
  return ROAST_OK;
}

roast_status_t roast_embedding_fwd_multi(roast_t h, const int32_t* ids, int32_t ntables, const int64_t* idx,
                                         int64_t n, float* out, roast_stream_t stream) {
  if (!out && ntables > 0 && n > 0) return fail(ROAST_ERR_CONFIG, "null out");
  return embedding_multi(h, ids, ntables, idx, n, out, nullptr, stream);
}

roast_status_t roast_embedding_bwd_multi(roast_t h, const int32_t* ids, int32_t ntables, const int64_t* idx,
                                         int64_t n, const float* dOut, roast_stream_t stream) {
  if (!dOut && ntables > 0 && n > 0) return fail(ROAST_ERR_CONFIG, "null dOut");
  return embedding_multi(h, ids, ntables, idx, n, nullptr, dOut, stream);
}

roast_status_t roast_set_autotune(roast_t h, roast_autotune_t strategy) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (strategy < ROAST_TUNE_OFF || strategy > ROAST_TUNE_TRAINING) return fail(ROAST_ERR_CONFIG, "bad strategy");
  if (c->autotune != int(strategy)) c->tuned.clear();
  c->autotune = int(strategy);
  return ROAST_OK;
}

roast_status_t roast_set_tuned(roast_t h, int32_t id, int32_t kernel, int64_t tokens, int32_t wm, int32_t splits) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, id, kLinear, &m);
  if (st) return st;
  if (kernel < 0 || kernel > 2 || wm < 1 || wm > 2 || splits < 1 || splits > 64 || tokens < 0 ||
      (kernel < 2 && splits != 1 && splits != 3 && splits != 4))
    return fail(ROAST_ERR_CONFIG, "bad tuned configuration");
  c->tuned[std::array<int64_t, 4>{kernel, m->H, m->O, tokens}] = {wm, splits};
  return ROAST_OK;
}

roast_status_t roast_get_tuned(roast_t h, int32_t id, int32_t kernel, int64_t tokens, int32_t* wm, int32_t* splits) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, id, kLinear, &m);
  if (st) return st;
  auto it = c->tuned.find(std::array<int64_t, 4>{kernel, m->H, m->O, tokens});
  if (it == c->tuned.end()) return fail(ROAST_ERR_STATE, "shape not tuned");
  if (wm) *wm = it->second.first;
  if (splits) *splits = it->second.second;
  return ROAST_OK;
}

roast_status_t roast_zero_grad(roast_t h, roast_stream_t stream) {
  Ctx* c = ctx(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  ROAST_CUDA_CHECK(cudaMemsetAsync(c->dM, 0, c->mem_size * sizeof(float), reinterpret_cast<cudaStream_t>(stream)));
  return ROAST_OK;
}

roast_status_t roast_sync_shadow(roast_t h, roast_stream_t stream) {
  Ctx* c = ctx(h);
  if (!c || !c->M || !c->shadow) return fail(ROAST_ERR_STATE, "not bound");
  ROAST_CUDA_CHECK(launch_sync_shadow(c, reinterpret_cast<cudaStream_t>(stream)));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_sgd_step(roast_t h, float lr, roast_stream_t stream) {
  Ctx* c = ctx(h);
  if (!c || !c->M || !c->shadow) return fail(ROAST_ERR_STATE, "not bound");
  ROAST_CUDA_CHECK(launch_optimizer(c, ROAST_OPT_SGD, lr, 0.f, 0.f, 0.f, 0.f, 1, 0, false,
                                    reinterpret_cast<cudaStream_t>(stream)));
  c->launches++;
  return ROAST_OK;
}


roast_status_t roast_optimizer_step(roast_t h, const roast_opt_config_t* cfg, int64_t step, roast_stream_t stream) {
  Ctx* c = ctx(h);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (roast_status_t st = opt_prepare(c, cfg, step, cfg && cfg->touched_only, s)) return st;
  ROAST_CUDA_CHECK(launch_optimizer(c, cfg->kind, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay, step,
                                    cfg->zero_grad, cfg->touched_only != 0, s));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_get_error(roast_t h) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  int32_t v = 0;
  cudaError_t e = cudaMemcpy(&v, c->d_err, sizeof(v), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "read error flag");
  if (v & 2) return fail(ROAST_ERR_STATE, "p2p exchange: a peer did not post within 20 s (sticky)");
  if (v & 4)
    return fail(ROAST_ERR_STATE, "chained GEMM: a ready-counter wait timed out (grid not co-resident?); "
                                 "its outputs are invalid (sticky)");
  if (v) return fail(ROAST_ERR_BOUNDS, "embedding index out of range (sticky)");
  return ROAST_OK;
}

roast_status_t roast_debug_tile_map(roast_t h, int32_t id, int64_t* off_host, int8_t* sgn_host) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (id < 0 || id >= int32_t(c->modules.size()) || c->modules[id].kind != kLinear)
    return fail(ROAST_ERR_STATE, "not a linear module");
  Module& m = c->modules[id];
  const int64_t nt = int64_t(m.nx) * m.ny;
  // read back the DEVICE copy the kernels use
  if (off_host) ROAST_CUDA_CHECK(cudaMemcpy(off_host, m.d_off, nt * sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (sgn_host) ROAST_CUDA_CHECK(cudaMemcpy(sgn_host, m.d_sgn, nt * sizeof(int8_t), cudaMemcpyDeviceToHost));
  return ROAST_OK;
}

roast_status_t roast_debug_chunk_map(roast_t h, int32_t id, const int64_t* rows, int64_t n, int64_t* off,
                                     int8_t* sgn, roast_stream_t stream) {
  Ctx* c = ctx(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (id < 0 || id >= int32_t(c->modules.size()) || c->modules[id].kind != kEmbedding)
    return fail(ROAST_ERR_STATE, "not an embedding module");
  ROAST_CUDA_CHECK(launch_chunk_map(c, c->modules[id], rows, n, off, sgn, reinterpret_cast<cudaStream_t>(stream)));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_debug_materialize(roast_t h, int32_t id, roast_dtype_t dt, void* W, roast_stream_t stream) {
  Ctx* c = ctx(h);
  Module* m;
  roast_status_t st = get_module(c, id, kLinear, &m);
  if (st) return st;
  ROAST_CUDA_CHECK(launch_materialize(c, *m, dt, W, reinterpret_cast<cudaStream_t>(stream)));
  c->launches++;
  return ROAST_OK;
}

roast_status_t roast_debug_opt_state(roast_t h, int32_t which, float* out_host) {
  Ctx* c = ctx(h);
  if (!c || !c->M) return fail(ROAST_ERR_STATE, "not bound");
  const float* src = which == 0 ? c->opt_s1 : which == 1 ? c->opt_s2 : nullptr;
  if (!src) return fail(ROAST_ERR_STATE, "optimizer state not allocated");
  if (!out_host) return fail(ROAST_ERR_CONFIG, "null output");
  ROAST_CUDA_CHECK(cudaDeviceSynchronize());
  ROAST_CUDA_CHECK(cudaMemcpy(out_host, src, size_t(c->mem_size) * sizeof(float), cudaMemcpyDeviceToHost));
  return ROAST_OK;
}

roast_status_t roast_lms_segments(const int64_t* sizes, int32_t n, int64_t mem_size, int32_t align,
                                  int64_t* seg_base, int64_t* seg_size) {
  if (!sizes || !seg_base || !seg_size || n < 1 || mem_size < 1 || align < 1)
    return fail(ROAST_ERR_CONFIG, "lms_segments: bad arguments");
  __int128 total = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (sizes[i] < 1) return fail(ROAST_ERR_CONFIG, "lms_segments: module sizes must be >= 1");
    total += sizes[i];
  }
  int64_t base = 0;
  for (int32_t i = 0; i < n; ++i) {
    // |M_i| = floor(f_i |M|), f_i = n_i / n, aligned down to A; the last piece takes the rest
    const int64_t size = i + 1 == n ? mem_size - base
                                    : int64_t((__int128(sizes[i]) * mem_size) / total) / align * align;
    seg_base[i] = base;
    seg_size[i] = size;
    base += size;
  }
  return ROAST_OK;
}

int64_t roast_launch_count(roast_t h) {
  Ctx* c = ctx(h);
  return c ? c->launches : -1;
}

}  // extern "C"

extern "C" roast_status_t roast_debug_hash_host(uint64_t seed, int32_t module, const uint64_t* keys, int64_t n,
                                                int64_t mem_size, int64_t span, int32_t align, int32_t use_sign,
                                                int64_t* off_out, int8_t* sgn_out) {
  if (!keys || n < 0 || span <= 0 || align <= 0) return fail(ROAST_ERR_CONFIG, "bad arguments");
  if (span > mem_size) return fail(ROAST_ERR_GEOMETRY, "span larger than |M|");
  ModuleHash h;
  h.off = make_coef(seed, uint32_t(module), 0);
  h.sgn = make_coef(seed, uint32_t(module), 1);
  h.set_range(uint64_t((mem_size - span) / align + 1));
  h.align = uint32_t(align);
  h.use_sign = use_sign ? 1u : 0u;
  for (int64_t i = 0; i < n; ++i) {
    if (keys[i] >= (uint64_t(1) << 60)) return fail(ROAST_ERR_CONFIG, "key >= 2^60");
    if (off_out) off_out[i] = int64_t(h.offset(keys[i]));
    if (sgn_out) sgn_out[i] = int8_t(h.sign(keys[i]));
  }
  return ROAST_OK;
}
