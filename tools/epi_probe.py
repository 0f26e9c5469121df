"""Diagnostics for the update kernel (SPHEMU_TC_DBG modes; a diagnostics build,
make -C paper_2408_04440_b200/csrc DIAG=1 -B): factor a strongly
diagonally dominant matrix, which stays positive definite even when a
diagnostic mode skips parts of the C epilogue, and print the busy time of the
dominant update class (tools/epi_probe.py N VARIANT HP_FORMAT)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, v, hp = int(sys.argv[1]), sys.argv[2], sys.argv[3]
cls = "update_sp" if v == "dpsp" else "update_hp"
a = torch.full((n, n), 1e-3, dtype=torch.float64, device="cuda")
a.diagonal().fill_(float(n))
h = sph.Cholesky(n, v, tile_size=512, hp_format=hp)
h.set_profiling(True, phases=[cls])
for it in range(3):
    h.load(a.data_ptr(), where=sph._sphemu.DEVICE, lda=n)
    if it == 2:
        h.reset_phase_times()
    h.factor()
    st = h.wait()
ph = h.phase_times()[cls]
fl = h.class_update_flops()[cls[-2:]]
print(f"dbg={os.environ.get('SPHEMU_TC_DBG', '0')} cg={os.environ.get('SPHEMU_TC_CG', '1')} n={n} {v}/{hp}: "
      f"factor {st.device_ms:.1f} ms, {cls} busy {ph['ms']:.1f} ms over {ph['launches']} launches "
      f"-> {fl / ph['ms'] / 1e9:.0f} TFLOP/s")
