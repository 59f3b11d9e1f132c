// placeholder until the tcgen05 kernels land: report UNSUPPORTED so the bf16
// path runs the SIMT kernels.
#include "roast_internal.h"
namespace roast {
roast_status_t sm100_prepare(Ctx*) { return ROAST_ERR_UNSUPPORTED; }
roast_status_t sm100_fwd(Ctx*, const Module&, const void*, void*, int64_t, cudaStream_t) { return ROAST_ERR_UNSUPPORTED; }
roast_status_t sm100_dx(Ctx*, const Module&, const void*, void*, int64_t, cudaStream_t) { return ROAST_ERR_UNSUPPORTED; }
roast_status_t sm100_dw(Ctx*, const Module&, const void*, const void*, int64_t, cudaStream_t) { return ROAST_ERR_UNSUPPORTED; }
}
