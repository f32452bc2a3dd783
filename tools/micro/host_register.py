"""Cost of pinning a pageable buffer in place (cudaHostRegister) against
staging it through pinned memory with memcpy, and the H2D rate from each."""
import ctypes as C
import time

import numpy as np
import torch

cudart = C.CDLL("libcudart.so.12") if False else None
torch.cuda.init()
lib = C.CDLL(torch.cuda.__file__.replace("cuda/__init__.py", "lib/libtorch_cuda.so"))
rt = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        rt = C.CDLL(name)
        break
    except OSError:
        pass
if rt is None:
    import glob, os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    rt = C.CDLL(cands[0])
nbytes = 1 << 30
a = np.ones(nbytes // 8)
d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
pin = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
for rep in range(2):
    t0 = time.perf_counter()
    rc = rt.cudaHostRegister(C.c_void_p(a.ctypes.data), C.c_size_t(nbytes), 0)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rc2 = rt.cudaMemcpy(C.c_void_p(d.data_ptr()), C.c_void_p(a.ctypes.data), C.c_size_t(nbytes), 1)
    t3 = time.perf_counter()
    rt.cudaHostUnregister(C.c_void_p(a.ctypes.data))
    t4 = time.perf_counter()
    print(f"register 1 GiB: {t1 - t0:.4f} s (rc {rc}), H2D from it {nbytes / (t3 - t2) / 1e9:.1f} GB/s "
          f"(rc {rc2}), unregister {t4 - t3:.4f} s")
    t0 = time.perf_counter()
    pin.numpy()[:] = a
    t1 = time.perf_counter()
    d.copy_(pin, non_blocking=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"memcpy to pinned (1 thread): {nbytes / (t1 - t0) / 1e9:.1f} GB/s, H2D pinned {nbytes / (t2 - t1) / 1e9:.1f} GB/s")
    t0 = time.perf_counter()
    rc2 = rt.cudaMemcpy(C.c_void_p(d.data_ptr()), C.c_void_p(a.ctypes.data), C.c_size_t(nbytes), 1)
    t1 = time.perf_counter()
    print(f"H2D pageable (driver staging): {nbytes / (t1 - t0) / 1e9:.1f} GB/s")
