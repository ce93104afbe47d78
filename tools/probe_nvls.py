"""Probe multicast (NVLS) support and handle types on the box's GPUs."""
from cuda.bindings import driver as d

def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1:] if isinstance(r, tuple) and len(r) > 1 else None

chk(d.cuInit(0))
n = chk(d.cuDeviceGetCount())[0]
for i in range(n):
    dev = chk(d.cuDeviceGet(i))[0]
    out = {}
    for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"):
        try:
            out[name.replace("CU_DEVICE_ATTRIBUTE_", "")] = chk(d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, name), dev))[0]
        except Exception as e:
            out[name] = f"error {e}"
    print(i, out, flush=True)
# granularity of a multicast object over all devices
prop = d.CUmulticastObjectProp()
prop.numDevices = n
prop.size = 2 << 20
prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
try:
    g = chk(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))[0]
    print("multicast granularity (recommended)", g)
    ctx = chk(d.cuDevicePrimaryCtxRetain(chk(d.cuDeviceGet(0))[0]))[0]
    chk(d.cuCtxSetCurrent(ctx))
    prop.size = g
    h = chk(d.cuMulticastCreate(prop))[0]
    print("cuMulticastCreate ok", h)
except Exception as e:
    print("multicast:", e)
