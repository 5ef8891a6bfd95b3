"""Development probe: does this GPU / driver offer NVLS multicast objects?
Creates a 1-device multicast object, binds a buffer, maps the multicast VA and
checks that a store through it lands in the buffer."""
import sys
import torch
from cuda.bindings import driver as drv

torch.cuda.init()
torch.zeros(1, device="cuda")
dev = 0


def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) == 2 else (r[1:] if isinstance(r, tuple) else None)


sup = ok(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
print("MULTICAST_SUPPORTED", sup)
if not sup:
    sys.exit(0)
mc = None
for ht in (0, drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
           drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC):
    prop = drv.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.handleTypes = int(ht)
    prop.size = 2 << 20
    for gflag in (drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM,
                  drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED):
        r = drv.cuMulticastGetGranularity(prop, gflag)
        print("handle", int(ht), "gran", gflag, r)
    gran = r[1] if r[0] == drv.CUresult.CUDA_SUCCESS else (2 << 20)
    size = ((2 << 20) + gran - 1) // gran * gran
    prop.size = size
    r = drv.cuMulticastCreate(prop)
    print("create", int(ht), size, r[0])
    if r[0] == drv.CUresult.CUDA_SUCCESS:
        mc = r[1]
        break
if mc is None:
    sys.exit(0)
ok(drv.cuMulticastAddDevice(mc, dev))
ap = drv.CUmemAllocationProp()
ap.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
ap.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
ap.location.id = dev
ap.requestedHandleTypes = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
mg = ok(drv.cuMemGetAllocationGranularity(ap, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
size = max(size, (size + mg - 1) // mg * mg)
mem = ok(drv.cuMemCreate(size, ap, 0))
ok(drv.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
uc = ok(drv.cuMemAddressReserve(size, 0, 0, 0))
ok(drv.cuMemMap(uc, size, 0, mem, 0))
mcva = ok(drv.cuMemAddressReserve(size, 0, 0, 0))
ok(drv.cuMemMap(mcva, size, 0, mc, 0))
acc = drv.CUmemAccessDesc()
acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
acc.location.id = dev
acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
ok(drv.cuMemSetAccess(uc, size, [acc], 1))
ok(drv.cuMemSetAccess(mcva, size, [acc], 1))
print("multicast VA", hex(int(mcva)), "unicast VA", hex(int(uc)), "size", size)
