"""Times the one-shot sphemu_gpu_tiled_cholesky_dense call (pinned host in and
out) and checks its output against the device-resident handle's factor."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, b = int(sys.argv[1]), int(sys.argv[2])
v = sys.argv[3] if len(sys.argv) > 3 else "dpsp"
pinned = (sys.argv[4] if len(sys.argv) > 4 else "pinned") == "pinned"
lib = sph._sphemu.lib()
h = sph.Cholesky(n, v, tile_size=b)
h.generate_spd(1)
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
h.store(a.data_ptr())
a += torch.tril(a, -1).T
h.load(a.data_ptr(), where=sph._sphemu.DEVICE, lda=n)
h.factor()
h.wait()
ref = torch.empty((n, n), dtype=torch.float64, device="cuda")
h.store(ref.data_ptr())
del h
ah = torch.empty((n, n), dtype=torch.float64, pin_memory=pinned)
fh = torch.empty((n, n), dtype=torch.float64, pin_memory=pinned)
ah.copy_(a)
del a
torch.cuda.synchronize()
cfg = sph._sphemu.make_config(v, b)
st = sph._sphemu.CholStats()
failed = C.c_int(-1)
for rep in range(4):
    fh.fill_(float("nan"))
    t0 = time.perf_counter()
    rc = lib.sphemu_gpu_tiled_cholesky_dense(C.c_void_p(ah.data_ptr()), 0, n, C.byref(cfg),
                                             C.c_void_p(fh.data_ptr()), 0, C.byref(st), C.byref(failed))
    dt = time.perf_counter() - t0
    assert rc == 0, rc
    same = torch.equal(fh.cuda(), ref)
    print(f"n={n} b={b} {v} {'pinned' if pinned else 'pageable'}: {dt*1e3:.1f} ms  {n**3/3/dt/1e12:.1f} TFLOP/s  "
          f"device {st.device_ms:.1f} ms  bitwise-equal={same}", flush=True)
lib.sphemu_gpu_release_cache()
