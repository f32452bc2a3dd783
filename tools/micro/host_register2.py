"""cudaHostRegister of fresh (touched) pageable memory in 128 MB chunks:
sequential and from 4 / 8 host threads at once."""
import ctypes as C
import glob
import os
import threading
import time

import numpy as np
import torch

torch.cuda.init()
rt = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        rt = C.CDLL(name)
        break
    except OSError:
        pass
if rt is None:
    rt = C.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))[0])
CH = 128 << 20
for threads in (1, 4, 8, 16):
    a = np.empty((4 << 30) // 8)
    a[:] = 1.0  # touched, like a std::vector's zero fill
    base = a.ctypes.data
    n = a.nbytes // CH
    t0 = time.perf_counter()
    def work(ids):
        for i in ids:
            rc = rt.cudaHostRegister(C.c_void_p(base + i * CH), C.c_size_t(CH), 0)
            assert rc == 0, rc
    ths = [threading.Thread(target=work, args=(range(t, n, threads),)) for t in range(threads)]
    for t in ths: t.start()
    for t in ths: t.join()
    t1 = time.perf_counter()
    for i in range(n):
        rt.cudaHostUnregister(C.c_void_p(base + i * CH))
    t2 = time.perf_counter()
    print(f"threads {threads}: register 4 GiB fresh in 128 MB chunks {a.nbytes / (t1 - t0) / 1e9:.1f} GB/s, unregister {a.nbytes / (t2 - t1) / 1e9:.1f} GB/s")
    del a
# memcpy rate with 16 threads into pinned
pin = torch.empty((1 << 30) // 8, dtype=torch.float64, pin_memory=True).numpy()
a = np.ones((1 << 30) // 8)
def cp(lo, hi):
    pin[lo:hi] = a[lo:hi]
for threads in (1, 4, 8, 16):
    t0 = time.perf_counter()
    step = a.size // threads
    ths = [threading.Thread(target=cp, args=(i * step, (i + 1) * step)) for i in range(threads)]
    for t in ths: t.start()
    for t in ths: t.join()
    t1 = time.perf_counter()
    print(f"memcpy 1 GiB to pinned, {threads} threads: {a.nbytes / (t1 - t0) / 1e9:.1f} GB/s")
