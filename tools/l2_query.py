import torch
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size / 2**20, "MB")
from cuda.bindings import runtime as rt
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0); print("max persisting L2", v / 2**20, "MB")
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0); print("max window", v / 2**20, "MB")
