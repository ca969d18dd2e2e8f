"""Does this box expose NVLink SHARP multicast objects?  Single process, all
visible GPUs: attribute, granularity, create + add devices + bind + map.
Prints one JSON line.  (Diagnostic for the NVLS barrier.)"""
import json

from cuda.bindings import driver as cu


def ok(r):
    return r[0] if isinstance(r, tuple) else r


def main():
    out = {}
    cu.cuInit(0)
    n = ok(cu.cuDeviceGetCount()[1:]) if False else cu.cuDeviceGetCount()[1]
    out["gpus"] = n
    devs = [cu.cuDeviceGet(i)[1] for i in range(n)]
    out["multicast_supported"] = [cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d)[1]
                                  for d in devs]
    ctxs = [cu.cuDevicePrimaryCtxRetain(d)[1] for d in devs]
    cu.cuCtxSetCurrent(ctxs[0])
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = n
    prop.size = 2 << 20
    prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    err, gran = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    out["granularity"] = [str(err), int(gran) if err == cu.CUresult.CUDA_SUCCESS else None]
    err, mc = cu.cuMulticastCreate(prop)
    out["create"] = str(err)
    if err == cu.CUresult.CUDA_SUCCESS:
        out["add_device"] = [str(cu.cuMulticastAddDevice(mc, d)[0]) for d in devs]
        binds = []
        for i, d in enumerate(devs):
            cu.cuCtxSetCurrent(ctxs[i])
            ap = cu.CUmemAllocationProp()
            ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
            ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            ap.location.id = i
            ap.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
            e2, h = cu.cuMemCreate(2 << 20, ap, 0)
            binds.append([str(e2), str(cu.cuMulticastBindMem(mc, 0, h, 0, 2 << 20, 0)[0])])
        out["bind"] = binds
    print(json.dumps(out))


if __name__ == "__main__":
    main()
