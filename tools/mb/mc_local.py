"""Step-by-step probe of a one-GPU multicast object through the CUDA driver API (cuda-python)."""
import torch
from cuda.bindings import driver as cu
torch.cuda.init(); torch.zeros(1, device="cuda")
print("init", cu.cuInit(0))
dev = cu.cuDeviceGet(0)[1]
print("mc attr", cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
for ht in (0, 1):
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.handleTypes = ht
    prop.size = 2 << 20
    r = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    print("ht", ht, "gran", r)
    if r[0] != cu.CUresult.CUDA_SUCCESS:
        continue
    prop.size = max(prop.size, r[1])
    r2 = cu.cuMulticastCreate(prop)
    print("create", r2[0])
    if r2[0] == cu.CUresult.CUDA_SUCCESS:
        print("add", cu.cuMulticastAddDevice(r2[1], dev))
