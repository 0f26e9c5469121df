"""Host-visible breakdown of one tiled_cholesky_dense call with pinned buffers."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, b = int(sys.argv[1]), int(sys.argv[2])
h = sph.Cholesky(n, "dpsp", tile_size=b)
h.generate_spd(1)
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
h.store(a.data_ptr())
a += torch.tril(a, -1).T
ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
fh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
ah.copy_(a)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    h2 = sph.Cholesky(n, "dpsp", tile_size=b)
    t1 = time.perf_counter()
    h2.load(ah.numpy())
    t2 = time.perf_counter()
    h2.factor()
    st = h2.wait()
    t3 = time.perf_counter()
    lib = sph._sphemu.lib()
    import ctypes as C
    lib.sphemu_gpu_chol_store_dense(h2.h, C.c_void_p(fh.data_ptr()), 0, n)
    t4 = time.perf_counter()
    del h2
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  load(H2D+tile) {1e3*(t2-t1):.1f}  factor {1e3*(t3-t2):.1f} "
          f"(dev {st.device_ms:.1f})  store(D2H) {1e3*(t4-t3):.1f}  destroy {1e3*(t5-t4):.1f}", flush=True)
