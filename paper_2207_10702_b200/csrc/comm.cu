// comm.cu — a6: data-parallel dM all-reduce over NCCL (NVLink 5 / NVSwitch).
//
// Under GMS every layer accumulates into the same dM, so the
// exchange is ONE in-place fp32 sum of |M| elements per step, issued on the
// compute stream after the last backward call.  libnccl.so.2
// is resolved at run time (the copy torch already loaded, if any) so the
// library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include "roast_internal.h"

namespace roast {
namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  if (a.loaded) return a;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return a;
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(lib, "ncclCommInitRank"));
  a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(lib, "ncclAllReduce"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(lib, "ncclCommDestroy"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(lib, "ncclGetErrorString"));
  a.loaded = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.CommDestroy && a.GetErrorString;
  return a;
}

roast_status_t nccl_fail(ncclResult_t r, const char* what) {
  return fail(ROAST_ERR_NCCL, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace

void comm_destroy(Ctx* c) {
  if (c->nccl_comm && api().loaded) api().CommDestroy(reinterpret_cast<ncclComm_t>(c->nccl_comm));
  c->nccl_comm = nullptr;
}

}  // namespace roast

using namespace roast;

extern "C" {

roast_status_t roast_comm_unique_id(uint8_t id_out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  if (!id_out) return fail(ROAST_ERR_CONFIG, "null id");
  if (!api().loaded) return fail(ROAST_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId uid;
  ncclResult_t r = api().GetUniqueId(&uid);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id_out, &uid, 128);
  return ROAST_OK;
}

roast_status_t roast_comm_init(roast_t h, int32_t rank, int32_t world, const uint8_t id[128]) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c) return fail(ROAST_ERR_STATE, "null handle");
  if (world < 1 || rank < 0 || rank >= world) return fail(ROAST_ERR_CONFIG, "bad rank / world");
  comm_destroy(c);
  c->rank = rank;
  c->world = world;
  if (world == 1 && !id) return ROAST_OK;   // single rank, no communicator (exchange is a no-op)
  if (!id) return fail(ROAST_ERR_CONFIG, "null id");
  // deterministic mode: a fixed all-reduce algorithm keeps the cross-rank summation order the
  // same run to run (NCCL_ALGO=Ring); a value the user set is kept
  if (c->cfg.deterministic) setenv("NCCL_ALGO", "Ring", 0);
  if (!api().loaded) return fail(ROAST_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t comm;
  ncclResult_t r = api().CommInitRank(&comm, world, uid, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  c->nccl_comm = comm;
  return ROAST_OK;
}

roast_status_t roast_grad_allreduce(roast_t h, roast_stream_t stream) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  if (!c->nccl_comm) {
    if (c->world == 1) return ROAST_OK;
    return fail(ROAST_ERR_STATE, "roast_comm_init has not been called");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  bool touched = false;
  if (c->exchange_mode != ROAST_EXCHANGE_DENSE) {
    // the interval tables are built on the first (eager) call; under graph capture they must exist
    if (!(c->touched_valid && c->touched_for == int64_t(c->modules.size()))) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        return fail(ROAST_ERR_STATE, "touched-set exchange: call roast_touched_size (or one eager exchange) "
                                     "before capturing");
      if (roast_status_t st = touched_prepare(c, s)) return st;
    }
    touched = c->exchange_mode == ROAST_EXCHANGE_TOUCHED || 2 * c->touched_n <= c->mem_size;
  }
  if (!touched) {
    ncclResult_t r = api().AllReduce(c->dM, c->dM, size_t(c->mem_size), ncclFloat32, ncclSum,
                                     reinterpret_cast<ncclComm_t>(c->nccl_comm), s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    return ROAST_OK;
  }
  if (c->touched_n == 0) return ROAST_OK;
  ROAST_CUDA_CHECK(launch_pack(c, 0, 1.f, s));
  ncclResult_t r = api().AllReduce(c->d_pack, c->d_pack, size_t(c->touched_n), ncclFloat32, ncclSum,
                                   reinterpret_cast<ncclComm_t>(c->nccl_comm), s);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(touched)");
  ROAST_CUDA_CHECK(launch_pack(c, 1, 1.f, s));
  c->launches += 2;
  return ROAST_OK;
}

roast_status_t roast_grad_exchange_step(roast_t h, const roast_opt_config_t* cfg, int64_t step,
                                        roast_stream_t stream) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  if (!c->nccl_comm && c->world > 1) return fail(ROAST_ERR_STATE, "roast_comm_init has not been called");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool want_touched = cfg && (cfg->touched_only || c->exchange_mode != ROAST_EXCHANGE_DENSE);
  if (roast_status_t st = opt_prepare(c, cfg, step, want_touched, s)) return st;
  const bool touched = cfg->touched_only || (c->exchange_mode == ROAST_EXCHANGE_TOUCHED) ||
                       (c->exchange_mode == ROAST_EXCHANGE_AUTO && 2 * c->touched_n <= c->mem_size);
  const ncclComm_t comm = reinterpret_cast<ncclComm_t>(c->nccl_comm);
  if (!touched) {   // dense: the in-place sum, then one pass over |M|
    if (comm) {
      ncclResult_t r = api().AllReduce(c->dM, c->dM, size_t(c->mem_size), ncclFloat32, ncclSum, comm, s);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    }
    ROAST_CUDA_CHECK(launch_optimizer(c, cfg->kind, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay,
                                      step, cfg->zero_grad, false, s));
    c->launches++;
    return ROAST_OK;
  }
  // touched: pack -> sum of the packed buffer -> the update reads the summed gradient straight
  // from the packed buffer (no unpack pass) and zeroes dM on the touched slots
  if (c->touched_n == 0) return ROAST_OK;
  ROAST_CUDA_CHECK(launch_pack(c, 0, 1.f, s));
  c->launches++;
  if (comm) {
    ncclResult_t r = api().AllReduce(c->d_pack, c->d_pack, size_t(c->touched_n), ncclFloat32, ncclSum, comm, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(touched)");
  }
  if (!cfg->zero_grad) {   // keep the documented dM contents (the summed gradient) when dM is not zeroed
    ROAST_CUDA_CHECK(launch_pack(c, 1, 1.f, s));
    c->launches++;
  }
  ROAST_CUDA_CHECK(launch_optimizer(c, cfg->kind, cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay, step,
                                    cfg->zero_grad, true, s, c->d_pack));
  c->launches++;
  return ROAST_OK;
}

}  // extern "C"
