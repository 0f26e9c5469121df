"""Device-resident timing of fit_var (var.cu) at the C2 size: L=180 (d=32 400
coefficients), T=1 000 daily steps, R=1, order 3. Algorithmic HBM bytes:
series read twice (16 B/element) + residuals written (8 B/row element)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

lib = sph._sphemu.lib()
R, T, d = 1, 1000, 180 * 180
for order in (1, 3):
    c = torch.randn(R, T, d, dtype=torch.float64, device="cuda") * 0.1
    c = torch.cumsum(c, dim=1) * 0.5
    res = torch.empty(R * (T - order), d, dtype=torch.float64, device="cuda")
    phi = torch.empty(order * d, dtype=torch.float64).numpy()
    se = torch.empty(order * d, dtype=torch.float64).numpy()
    zc, uc, nrm = C.c_int64(), C.c_int64(), C.c_double()

    def call():
        rc = lib.sphemu_gpu_fit_var(C.c_void_p(c.data_ptr()), 1, R, T, d, order, C.c_void_p(phi.ctypes.data),
                                    C.c_void_p(se.ctypes.data), C.c_void_p(res.data_ptr()), 1, C.byref(zc),
                                    C.byref(uc), C.byref(nrm))
        assert rc == 0, lib.sphemu_gpu_last_error()

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        call()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    nbytes = 16 * R * T * d + 8 * R * (T - order) * d
    print(f"fit_var order={order}: {ms:.3f} ms per call, {nbytes / ms / 1e6:.0f} GB/s algorithmic, "
          f"unstable {uc.value} zeroed {zc.value}")
