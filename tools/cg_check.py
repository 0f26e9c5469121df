"""Factor once and print a digest of the factor (compare runs under
different SPHEMU_TC_* settings)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, b, v, hp = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
h = sph.Cholesky(n, v, tile_size=b, hp_format=hp)
for _ in range(2):
    h.generate_spd(1)
    h.factor()
    st = h.wait()
out = torch.empty((n, n), dtype=torch.float64, device="cuda")
h.store(out.data_ptr())
dig = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"n={n} {v}/{hp} CG={os.environ.get('SPHEMU_TC_CG', '2')} {st.device_ms:.2f} ms "
      f"{n**3/3/st.device_ms/1e9:.1f} TFLOP/s probe={h.residual_probe(1, 2):.3e} sat={st.half_saturations} digest={dig}")
