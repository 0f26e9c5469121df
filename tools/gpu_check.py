"""Quick staged GPU sanity run (development aid): parity vs the oracle on
small cases, then timings. Usage: python tools/gpu_check.py [stage...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
import paper_2408_04440_b200 as sph  # noqa: E402

stages = sys.argv[1:] or ["chol64", "cholmp", "tensor", "sht", "time"]
TH = {"dp": 1e-12, "dpsp": 5e-6, "dpsphp": 1e-2, "dphp": 5e-2}


def p(*a):
    print(*a, flush=True)


if "chol64" in stages:
    for n in (96, 100):
        a = O.make_spd(n, 3)
        f, st = sph.tiled_cholesky(a, "dp", tile_size=32, compute="fp64")
        ref = O.dense_cholesky(a)
        p("fp64 dp n", n, "max|L-Lref|", np.abs(f - ref).max(), "resid", O.relative_residual(a, f))
    f, st = sph.tiled_cholesky(np.array([[4., 2.], [2., 3.]]), "dp", tile_size=1, compute="fp64")
    p("2x2", f.tolist())
    n = 96
    a = np.eye(n); a[40, 40] = -1
    try:
        sph.tiled_cholesky(a, "dp", tile_size=32, compute="fp64")
        p("ERROR no failure")
    except sph.NotPositiveDefiniteError as e:
        p("NotSPD tile", e.tile_index)

if "cholmp" in stages:
    a = O.make_spd(256, 5)
    for v in TH:
        f, st = sph.tiled_cholesky(a, v, tile_size=64, compute="fp64")
        ref, rst = O.tiled_cholesky(a, v, tile_size=64)
        p("fp64-compute", v, "resid gpu", O.relative_residual(a, f), "oracle", O.relative_residual(a, ref),
          "maxdiff", np.abs(f - ref).max())

if "tensor" in stages:
    for n, b in ((1024, 256), (1000, 128), (2048, 512)):
        a = O.make_spd(n, 5)
        for v in TH:
            t = time.time()
            f, st = sph.tiled_cholesky(a, v, tile_size=b)
            dt = time.time() - t
            ref, _ = O.tiled_cholesky(a, v, tile_size=b, workers=8)
            rg, ro = O.relative_residual(a, f), O.relative_residual(a, ref)
            p(f"tensor n={n} b={b} {v}: resid gpu {rg:.3e} oracle {ro:.3e} ok={rg <= max(2*ro, TH[v])} "
              f"maxdiff {np.abs(f-ref).max():.3e} {dt:.2f}s")

if "sht" in stages:
    for (nt, nphi, L) in ((9, 16, 8), (33, 64, 16), (46, 90, 45), (181, 360, 180)):
        P = O.Plan(nt, nphi, L)
        c = np.stack([O.draw_random_coefficients(L, s) for s in range(5)])
        fo = P.inverse(c)
        g = sph.ShtPlan(nt, nphi, L)
        fg = g.inverse(c)
        cg = g.forward(fo)
        co = P.forward(fo)
        p(f"sht {nt}x{nphi} L={L}: inv rel {np.abs(fg-fo).max()/np.abs(fo).max():.2e} "
          f"fwd rel {np.abs(cg-co).max()/np.abs(co).max():.2e} roundtrip {np.abs(cg-c).max():.2e} plan {g.plan_seconds:.3f}s")

if "time" in stages:
    for n, b, v in ((8192, 512, "dpsp"), (32400, 512, "dpsp")):
        h = sph.Cholesky(n, v, tile_size=b)
        f = h.flops()
        for rep in range(2):
            h.generate_spd(1)
            h.factor()
            st = h.wait()
        tf = n ** 3 / 3 / (st.device_ms * 1e-3) / 1e12
        p(f"time n={n} b={b} {v}: {st.device_ms:.1f} ms  {tf:.1f} TFLOP/s launches {st.launches} flops {f}")
    import torch
    for (nt, nphi, L, T) in ((181, 360, 180, 1000), (721, 1440, 720, 64)):
        g = sph.ShtPlan(nt, nphi, L, wigner_cap_bytes=8 << 30)
        coef = torch.randn(T, L * L, dtype=torch.float64, device="cuda")
        fld = torch.empty(T, nt, nphi, dtype=torch.float64, device="cuda")
        out = torch.empty_like(coef)
        for rep in range(3):
            torch.cuda.synchronize(); t = time.time()
            g.inverse_device(coef.data_ptr(), T, fld.data_ptr())
            torch.cuda.synchronize(); ti = time.time() - t
            t = time.time()
            g.forward_device(fld.data_ptr(), T, out.data_ptr())
            torch.cuda.synchronize(); tf_ = time.time() - t
        p(f"sht L={L} T={T}: plan {g.plan_seconds:.2f}s inv {T/ti:.0f} snap/s fwd {T/tf_:.0f} snap/s")
