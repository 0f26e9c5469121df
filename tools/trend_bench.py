"""Device-resident timing of the trend kernels (trend.cu) at the C4 grid
(721x1440 points, K=5 harmonics, hourly period): retrend of R x T standardized
fields and the mean table. Reports algorithmic HBM GB/s (16 B per element for
retrend, 8 B for the table) from CUDA events around the C-ABI calls."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

lib = sph._sphemu.lib()
points, K, period, T, R = 721 * 1440, 5, 8760, 96, 4
rec = np.random.default_rng(1).standard_normal((points, 5 + 2 * K))
rec[:, -1] = 1.0 + np.abs(rec[:, -1])
z = torch.randn(R, T, points, dtype=torch.float64, device="cuda")
out = torch.empty_like(z)
drec = torch.from_numpy(rec).cuda()  # device records: retrend reads them in place
tab = torch.empty(T, points, dtype=torch.float64, device="cuda")
vp = C.c_void_p


def retrend():
    rc = lib.sphemu_gpu_retrend(vp(z.data_ptr()), 1, R, T, vp(drec.data_ptr()), points, K, period, None, 0, None, 0,
                                1, vp(out.data_ptr()), 1)
    assert rc == 0, lib.sphemu_gpu_last_error()


def table():
    rc = lib.sphemu_gpu_mean_table(vp(rec.ctypes.data), points, K, period, None, 0, None, 0, T, 1,
                                   vp(tab.data_ptr()), 1)
    assert rc == 0, lib.sphemu_gpu_last_error()


for name, fn, nbytes in (("retrend", retrend, 16 * R * T * points), ("mean_table", table, 8 * T * points)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    print(f"{name}: {ms:.3f} ms per call (retrend: device records; mean_table: host records, {points * (5 + 2 * K) * 8 / 1e6:.0f} MB H2D), "
          f"{nbytes / ms / 1e6:.0f} GB/s algorithmic")
