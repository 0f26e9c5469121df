"""Plan-build time (Wigner tables + Legendre operators, all on the device) at
the C2 / C3 / C4 band limits."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2408_04440_b200 as sph

for nt, nphi, L in [(181, 360, 180), (361, 720, 360), (721, 1440, 720)]:
    for rep in range(2):
        t = time.perf_counter()
        p = sph.ShtPlan(nt, nphi, L, wigner_cap_bytes=8 << 30)
        wall = time.perf_counter() - t
        print(f"{nt}x{nphi} L={L} rep {rep}: plan {p.plan_seconds:.3f} s, wall {wall:.3f} s", flush=True)
        del p
