"""cudaHostRegister / cudaHostUnregister throughput on already-touched pageable memory (the
drop-in's inputs), 1-8 threads registering disjoint slices: is pinning the caller's arrays in place
cheaper than staging them through the pinned ring?"""
import ctypes
import threading
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so.12") if False else None
torch.cuda.init()
lib = ctypes.CDLL(torch.cuda.__file__.replace("cuda/__init__.py", "lib/libcudart.so.12")) if False else None
try:
    lib = ctypes.CDLL("libcudart.so.12")
except OSError:
    import glob
    import os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    lib = ctypes.CDLL(cands[0])
lib.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
lib.cudaHostUnregister.argtypes = [ctypes.c_void_p]
GB = 12
a = np.ones(GB << 27, dtype=np.float64)  # 12 GB, touched
base = a.ctypes.data
n = a.nbytes
for threads in (1, 4, 8, 16):
    part = (n // threads) & ~((1 << 21) - 1)
    spans = [(base + i * part, part if i < threads - 1 else n - i * part) for i in range(threads)]
    errs = []

    def reg(p, s):
        errs.append(lib.cudaHostRegister(ctypes.c_void_p(p), ctypes.c_size_t(s), 0))

    def unreg(p, s):
        errs.append(lib.cudaHostUnregister(ctypes.c_void_p(p)))

    t0 = time.perf_counter()
    ts = [threading.Thread(target=reg, args=sp) for sp in spans]
    [t.start() for t in ts]
    [t.join() for t in ts]
    t1 = time.perf_counter()
    ts = [threading.Thread(target=unreg, args=sp) for sp in spans]
    [t.start() for t in ts]
    [t.join() for t in ts]
    t2 = time.perf_counter()
    print(f"{threads:2d} threads: register {n / (t1 - t0) / 1e9:6.1f} GB/s, unregister {n / (t2 - t1) / 1e9:6.1f} GB/s, "
          f"errors {sorted(set(errs))}", flush=True)
