"""Probe multicast-object creation on this box (no kernels launched)."""
from cuda.bindings import driver as cu

cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
err, ctx = cu.cuDevicePrimaryCtxRetain(dev)
cu.cuCtxSetCurrent(ctx)
print("multicast attr", cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
for nd in (1, 2):
    for ht in ("CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC", "CU_MEM_HANDLE_TYPE_NONE"):
        p = cu.CUmulticastObjectProp()
        p.numDevices = nd
        p.size = 2 << 20
        p.handleTypes = getattr(cu.CUmemAllocationHandleType, ht)
        r = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        r2 = cu.cuMulticastCreate(p)
        print(nd, ht, "gran", r, "create", r2[0])
        if r2[0] == cu.CUresult.CUDA_SUCCESS:
            print("   add", cu.cuMulticastAddDevice(r2[1], dev))
            cu.cuMemRelease(r2[1])
