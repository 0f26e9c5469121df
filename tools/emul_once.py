"""One emulation from the tiled factor (for ncu captures): L = 180 (d = 32 400),
factor of the rho = 0.999 generator (dpsphp/bf16, b = 512), 100 replicates x 24
steps, AR(3), Philox, fields to HBM."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 180
variant = sys.argv[2] if len(sys.argv) > 2 else "dpsphp"
d = L * L
h = sph.Cholesky(d, variant, tile_size=512, hp_format="bf16")
h.generate_spd(1, rho=0.999)
h.factor()
h.wait()
nt, nphi = L + 1, 2 * L
plan = sph.ShtPlan(nt, nphi, L)
phi = np.stack([np.full(d, x) for x in (0.6, 0.25, 0.15)])
pts = nt * nphi
out = torch.empty((100, 24, nt, nphi), dtype=torch.float64, device="cuda")
for _ in range(2):
    h.emulate(plan, phi, np.zeros((24, pts)), np.ones(pts), np.full(pts, 0.04), 24, seed=7, r_len=100,
              out_ptr=out.data_ptr())
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
