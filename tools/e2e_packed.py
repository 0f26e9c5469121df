"""Host-buffer path timings under the current SPHEMU_PACKED_IO / SPHEMU_IO_THREADS
setting: load alone (H2D + tiling) and the one-shot tiled_cholesky_dense call."""
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
tag = f"packed={os.environ.get('SPHEMU_PACKED_IO', '1')} threads={os.environ.get('SPHEMU_IO_THREADS', 'default')}"
for rep in range(3):
    t0 = time.perf_counter()
    lib.sphemu_gpu_chol_load_dense(h.h, C.c_void_p(ah.data_ptr()), 0, n)
    print(f"{tag} load {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
del h
cfg = sph._sphemu.make_config("dpsp", b, lookahead=1)
st = sph._sphemu.CholStats()
ft = C.c_int()
for rep in range(3):
    t0 = time.perf_counter()
    rc = lib.sphemu_gpu_tiled_cholesky_dense(C.c_void_p(ah.data_ptr()), 0, n, C.byref(cfg), C.c_void_p(fh.data_ptr()), 0,
                                             C.byref(st), C.byref(ft))
    print(f"{tag} one-shot {1e3 * (time.perf_counter() - t0):.1f} ms rc={rc}", flush=True)
