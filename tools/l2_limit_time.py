import time
import torch
from cuda.bindings import runtime as rt
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
err, mx = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
for it in range(3):
    for v in (mx, 0):
        t0 = time.perf_counter()
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, v)
        t1 = time.perf_counter()
        print(f"set {v >> 20} MB: {1e3 * (t1 - t0):.3f} ms")
    t0 = time.perf_counter()
    rt.cudaCtxResetPersistingL2Cache()
    print(f"reset: {1e3 * (time.perf_counter() - t0):.3f} ms")
