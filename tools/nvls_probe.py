"""Which cuMulticastCreate properties does this box's driver accept?  (NVLS capability probe,
diagnostic only; the library's own probe is roast_nvls_supported / roast_nvls_create.)"""
from cuda.bindings import driver as d

print("cuInit", d.cuInit(0))
err, dev = d.cuDeviceGet(0)
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    a = getattr(d.CUdevice_attribute, attr, None)
    if a is not None:
        print(attr, d.cuDeviceGetAttribute(a, dev))
err, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
H = d.CUmemAllocationHandleType
for nd in (1, 2):
    for ht in (0, H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, H.CU_MEM_HANDLE_TYPE_FABRIC):
        p = d.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = ht
        p.size = 2 << 20
        e1, g = d.cuMulticastGetGranularity(p, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        p.size = max(g, 2 << 20)
        e2, mc = d.cuMulticastCreate(p)
        print(f"numDevices {nd} handleTypes {int(ht)} gran {e1} {g} -> create {e2}")
        if e2 == d.CUresult.CUDA_SUCCESS:
            print("  addDevice", d.cuMulticastAddDevice(mc, dev))
            d.cuMemRelease(mc)
