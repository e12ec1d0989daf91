import torch
p = torch.cuda.get_device_properties(0)
print("L2 bytes", p.L2_cache_size, "persisting max", torch.cuda.get_device_properties(0).__dict__ if False else "")
from cuda import cudart
for a in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrL2CacheSize"):
    err, v = cudart.cudaDeviceGetAttribute(getattr(cudart.cudaDeviceAttr, a), 0)
    print(a, v)
