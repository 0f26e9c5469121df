"""Component times of the host-buffer path (serialized): H2D+tile, factor, D2H by columns."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, b = 32400, 512
lib = sph._sphemu.lib()
h = sph.Cholesky(n, "dpsp", tile_size=b)
h.generate_spd(1)
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
h.store(a.data_ptr())
a += torch.tril(a, -1).T
ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
ah.copy_(a)
del a
fh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    lib.sphemu_gpu_chol_load_dense(h.h, C.c_void_p(ah.data_ptr()), 0, n)
    t1 = time.perf_counter()
    h.factor()
    h.wait()
    t2 = time.perf_counter()
    lib.sphemu_gpu_chol_store_dense(h.h, C.c_void_p(fh.data_ptr()), 0, n)
    t3 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.1f} ms  factor {1e3*(t2-t1):.1f} ms  store {1e3*(t3-t2):.1f} ms", flush=True)
t0 = time.perf_counter()
fh.zero_()
print(f"host zero of 8.4 GB (torch, 1 thread?): {1e3*(time.perf_counter()-t0):.1f} ms")
