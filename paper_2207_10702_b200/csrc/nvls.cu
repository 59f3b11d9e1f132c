// NVLS (NVSwitch multicast) variant of the dM exchange fused with the update (SURVEY.md §8(e),
// §8(f) NEXT #1; the exchange is a6 = P:194 "communication is directly proportional to model
// size", the update a7 = P:440 / P:749-813 `tab:total-opt`).
//
// The P2P exchange (p2p.cu) reads every peer's packed gradient over NVLink and sums the W
// copies on the SMs.  On an NVSwitch system the switch itself can reduce: the exchange window of
// every rank is bound to ONE multicast object, and
//   - multimem.ld_reduce.add.v4.f32 on the multicast alias of buffer[p] returns sum_r buffer_r[p],
//     reduced in the switch (one NVLink read per element instead of W - 1);
//   - multimem.st on the alias writes every rank's copy (the two-shot gather becomes a local read);
//   - the post / signal flags are written to every rank by one multimem.st.
// The kernels are the P2P ones (post, opt_kernel finish / reduce, signal2, gather) with those
// three substitutions; window layout, epochs and the double buffering are unchanged, so the
// whole exchange + optimizer + shadow refresh + dM zero stays two (one-shot) or four (two-shot)
// launches per step and graph-capturable.
//
// Set-up (all ranks, in this order; the Python binding drives it over torch.distributed):
//   roast_nvls_supported    capability probe (device attribute + driver entry points)
//   roast_nvls_create       rank 0: cuMulticastCreate for `world` devices, sized for the window;
//                           exports a POSIX file descriptor (sent to the peers over a unix socket)
//   roast_nvls_import       ranks != 0: import the object from that descriptor
//   roast_nvls_add_device   every rank adds its device; ALL ranks must return before any bind
//   roast_nvls_bind         allocate this rank's window memory (cuMemCreate), bind it, map the
//                           unicast and the multicast aliases; then a barrier before the first step
// A failure anywhere returns an error and leaves the handle on the P2P / NCCL paths (the binding
// falls back to the two-shot P2P exchange).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "roast_internal.h"

namespace roast {
namespace {

struct Drv {
  CUresult (*getAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*exportH)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*importH)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*memGran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static Drv d = [] {
    Drv x;
    x.ok = entry("cuDeviceGetAttribute", x.getAttr) && entry("cuMulticastGetGranularity", x.mcGran) &&
           entry("cuMulticastCreate", x.mcCreate) && entry("cuMulticastAddDevice", x.mcAddDevice) &&
           entry("cuMulticastBindMem", x.mcBindMem) && entry("cuMulticastUnbind", x.mcUnbind) &&
           entry("cuMemExportToShareableHandle", x.exportH) &&
           entry("cuMemImportFromShareableHandle", x.importH) &&
           entry("cuMemGetAllocationGranularity", x.memGran) && entry("cuMemCreate", x.memCreate) &&
           entry("cuMemRelease", x.memRelease) && entry("cuMemAddressReserve", x.addrReserve) &&
           entry("cuMemAddressFree", x.addrFree) && entry("cuMemMap", x.memMap) && entry("cuMemUnmap", x.memUnmap) &&
           entry("cuMemSetAccess", x.setAccess);
    return x;
  }();
  return d;
}

roast_status_t cu_fail(CUresult r, const char* what) {
  return fail(ROAST_ERR_CUDA, std::string(what) + " failed (CUresult " + std::to_string(int(r)) + ")");
}
#define ROAST_CU_CHECK(call)                       \
  do {                                             \
    CUresult _r = (call);                          \
    if (_r != CUDA_SUCCESS) return cu_fail(_r, #call); \
  } while (0)

Ctx* nctx(roast_t h) { return reinterpret_cast<Ctx*>(h); }

// window bytes for the current touched set (the p2p.cu layout: header | 2 packed buffers | M
// buffer), rounded up to the multicast and allocation granularities
roast_status_t window_size(Ctx* c, int world, size_t* out) {
  if (roast_status_t st = touched_prepare(c, 0)) return st;
  const int64_t n = (c->touched_n + 3) / 4 * 4;
  const size_t need = size_t(kP2PHeader + 3 * n * int64_t(sizeof(float)));
  CUmulticastObjectProp mp{};
  mp.numDevices = unsigned(world);
  mp.size = need;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g1 = 0, g2 = 0;
  ROAST_CU_CHECK(drv().mcGran(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->nvls_dev;
  ROAST_CU_CHECK(drv().memGran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t g = std::max(g1, g2);
  *out = (need + g - 1) / g * g;
  return ROAST_OK;
}

roast_status_t check_handle(Ctx* c) {
  if (!c || !c->dM) return fail(ROAST_ERR_STATE, "not bound");
  if (!drv().ok) return fail(ROAST_ERR_UNSUPPORTED, "NVLS: driver entry points unavailable");
  if (c->nvls_dev < 0) ROAST_CUDA_CHECK(cudaGetDevice(&c->nvls_dev));
  return ROAST_OK;
}

}  // namespace

void nvls_destroy(Ctx* c) {
  const Drv& d = drv();
  if (!d.ok) return;
  if (c->nvls_mc_va) {
    d.memUnmap(CUdeviceptr(c->nvls_mc_va), c->nvls_size);
    d.addrFree(CUdeviceptr(c->nvls_mc_va), c->nvls_size);
  }
  if (c->nvls_uc_va) {
    d.memUnmap(CUdeviceptr(c->nvls_uc_va), c->nvls_size);
    d.addrFree(CUdeviceptr(c->nvls_uc_va), c->nvls_size);
  }
  if (c->nvls_memb) d.mcUnbind(CUmemGenericAllocationHandle(c->nvls_mc), CUdevice(c->nvls_dev), 0, c->nvls_size);
  if (c->nvls_phys) d.memRelease(CUmemGenericAllocationHandle(c->nvls_phys));
  if (c->nvls_have_mc) d.memRelease(CUmemGenericAllocationHandle(c->nvls_mc));
  if (c->nvls_bound) {
    c->p2p_world = 0;
    c->p2p_bytes = c->p2p_n = 0;
  }
  c->nvls_mc = c->nvls_phys = c->nvls_uc_va = c->nvls_mc_va = 0;
  c->nvls_size = 0;
  c->nvls_world = 0;
  c->nvls_have_mc = c->nvls_added = c->nvls_memb = c->nvls_bound = false;
}

}  // namespace roast

using namespace roast;

extern "C" {

roast_status_t roast_nvls_supported(int32_t device, int32_t* supported) {
  if (!supported) return fail(ROAST_ERR_CONFIG, "null output");
  *supported = 0;
  const Drv& d = drv();
  if (!d.ok) return ROAST_OK;
  int v = 0;
  if (d.getAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, CUdevice(device)) != CUDA_SUCCESS) return ROAST_OK;
  *supported = v ? 1 : 0;
  return ROAST_OK;
}

roast_status_t roast_nvls_create(roast_t h, int32_t world, int32_t* fd) {
  Ctx* c = nctx(h);
  if (roast_status_t st = check_handle(c)) return st;
  if (world < 1 || world > kP2PMaxWorld || !fd) return fail(ROAST_ERR_CONFIG, "NVLS: 1 <= world <= 8, fd non-null");
  if (c->nvls_have_mc) return fail(ROAST_ERR_STATE, "NVLS: multicast object already created / imported");
  size_t size = 0;
  if (roast_status_t st = window_size(c, world, &size)) return st;
  CUmulticastObjectProp mp{};
  mp.numDevices = unsigned(world);
  mp.size = size;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mc;
  ROAST_CU_CHECK(drv().mcCreate(&mc, &mp));
  int f = -1;
  CUresult r = drv().exportH(&f, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) {
    drv().memRelease(mc);
    return cu_fail(r, "cuMemExportToShareableHandle");
  }
  c->nvls_mc = mc;
  c->nvls_have_mc = true;
  c->nvls_size = size;
  c->nvls_world = world;
  *fd = f;
  return ROAST_OK;
}

roast_status_t roast_nvls_import(roast_t h, int32_t world, int32_t fd) {
  Ctx* c = nctx(h);
  if (roast_status_t st = check_handle(c)) return st;
  if (world < 1 || world > kP2PMaxWorld || fd < 0) return fail(ROAST_ERR_CONFIG, "NVLS: 1 <= world <= 8, fd >= 0");
  if (c->nvls_have_mc) return fail(ROAST_ERR_STATE, "NVLS: multicast object already created / imported");
  size_t size = 0;
  if (roast_status_t st = window_size(c, world, &size)) return st;
  CUmemGenericAllocationHandle mc;
  ROAST_CU_CHECK(drv().importH(&mc, reinterpret_cast<void*>(uintptr_t(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  c->nvls_mc = mc;
  c->nvls_have_mc = true;
  c->nvls_size = size;
  c->nvls_world = world;
  return ROAST_OK;
}

roast_status_t roast_nvls_add_device(roast_t h) {
  Ctx* c = nctx(h);
  if (roast_status_t st = check_handle(c)) return st;
  if (!c->nvls_have_mc) return fail(ROAST_ERR_STATE, "NVLS: create or import the multicast object first");
  if (!c->nvls_added) {
    ROAST_CU_CHECK(drv().mcAddDevice(CUmemGenericAllocationHandle(c->nvls_mc), CUdevice(c->nvls_dev)));
    c->nvls_added = true;
  }
  return ROAST_OK;
}

namespace {
roast_status_t nvls_map(Ctx* c) {
  const Drv& d = drv();
  const size_t size = c->nvls_size;
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = c->nvls_dev;
  CUmemGenericAllocationHandle phys;
  ROAST_CU_CHECK(d.memCreate(&phys, size, &ap, 0));
  c->nvls_phys = phys;
  ROAST_CU_CHECK(d.mcBindMem(CUmemGenericAllocationHandle(c->nvls_mc), 0, phys, 0, size, 0));
  c->nvls_memb = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = c->nvls_dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcva = 0;
  ROAST_CU_CHECK(d.addrReserve(&uc, size, size, 0, 0));
  c->nvls_uc_va = uc;
  ROAST_CU_CHECK(d.memMap(uc, size, 0, phys, 0));
  ROAST_CU_CHECK(d.setAccess(uc, size, &acc, 1));
  ROAST_CU_CHECK(d.addrReserve(&mcva, size, size, 0, 0));
  c->nvls_mc_va = mcva;
  ROAST_CU_CHECK(d.memMap(mcva, size, 0, CUmemGenericAllocationHandle(c->nvls_mc), 0));
  ROAST_CU_CHECK(d.setAccess(mcva, size, &acc, 1));
  ROAST_CUDA_CHECK(cudaMemset(reinterpret_cast<void*>(uc), 0, size));   // flags and epoch start at 0 on every rank
  return ROAST_OK;
}
}  // namespace

roast_status_t roast_nvls_bind(roast_t h, int32_t rank) {
  Ctx* c = nctx(h);
  if (roast_status_t st = check_handle(c)) return st;
  if (!c->nvls_added) return fail(ROAST_ERR_STATE, "NVLS: roast_nvls_add_device on every rank first");
  if (c->nvls_bound) return ROAST_OK;
  if (rank < 0 || rank >= c->nvls_world) return fail(ROAST_ERR_CONFIG, "NVLS: 0 <= rank < world");
  if (roast_status_t st = nvls_map(c)) {   // undo everything: the handle stays on the P2P / NCCL paths
    nvls_destroy(c);
    return st;
  }
  // the window of the P2P kernels is now the unicast alias; every "peer" entry is this rank's
  // own window (peers are reached through the multicast alias instead)
  for (int r = 0; r < kP2PMaxWorld; ++r) {
    if (c->p2p_opened[r] && c->p2p_peer[r]) cudaIpcCloseMemHandle(c->p2p_peer[r]);
    c->p2p_opened[r] = false;
    c->p2p_peer[r] = nullptr;
  }
  cudaFree(c->p2p_win);
  c->p2p_win = reinterpret_cast<char*>(c->nvls_uc_va);
  c->p2p_bytes = int64_t(c->nvls_size);
  c->p2p_n = c->touched_n;
  c->p2p_rank = rank;
  c->p2p_world = c->nvls_world;
  for (int r = 0; r < c->nvls_world; ++r) c->p2p_peer[r] = c->p2p_win;
  c->nvls_bound = true;
  return ROAST_OK;
}

roast_status_t roast_nvls_reset(roast_t h) {
  Ctx* c = nctx(h);
  if (!c) return fail(ROAST_ERR_CONFIG, "null handle");
  if (c->nvls_bound) {   // back to a fresh (lazily allocated) P2P window
    for (int r = 0; r < kP2PMaxWorld; ++r) c->p2p_peer[r] = nullptr;
    c->p2p_win = nullptr;
  }
  nvls_destroy(c);
  return ROAST_OK;
}

roast_status_t roast_nvls_bound(roast_t h, int32_t* bound) {
  Ctx* c = nctx(h);
  if (!c || !bound) return fail(ROAST_ERR_CONFIG, "null handle / output");
  *bound = c->nvls_bound ? 1 : 0;
  return ROAST_OK;
}

}  // extern "C"
