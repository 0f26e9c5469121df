"""One warm forward+inverse SHT batch (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

nt, nphi, L, T = (int(x) for x in sys.argv[1:5])
g = sph.ShtPlan(nt, nphi, L, wigner_cap_bytes=8 << 30)
c = torch.randn(T, L * L, dtype=torch.float64, device="cuda")
f = torch.empty(T, nt, nphi, dtype=torch.float64, device="cuda")
o = torch.empty_like(c)
for _ in range(int(sys.argv[5]) if len(sys.argv) > 5 else 2):
    g.inverse_device(c.data_ptr(), T, f.data_ptr())
    g.forward_device(f.data_ptr(), T, o.data_ptr())
torch.cuda.synchronize()
print("round trip", (o - c).abs().max().item())
