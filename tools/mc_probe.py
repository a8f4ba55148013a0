"""Which multicast-object properties does this GPU accept (diagnostic)?"""
import torch
from cuda.bindings import driver as d

torch.zeros(1, device="cuda")
dev = d.cuDeviceGet(0)[1]
H = d.CUmemAllocationHandleType
for name, ht in (("none", 0), ("posix_fd", H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                 ("fabric", H.CU_MEM_HANDLE_TYPE_FABRIC)):
    mp = d.CUmulticastObjectProp()
    mp.numDevices = 1
    mp.handleTypes = ht
    mp.size = 2 << 20
    g = d.cuMulticastGetGranularity(mp, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    if g[0] == d.CUresult.CUDA_SUCCESS:
        mp.size = max(mp.size, g[1])
    r = d.cuMulticastCreate(mp)
    print(name, "gran", g, "create", r[0])
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    print(attr, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, attr), dev))
