"""DP-class trailing updates on the INT8 tensor cores (ozaki.cuh) against the
FP64 DMMA path (SPHEMU_DP_EMU=0): the same factorizations both ways.

Bounds: on make_spd_test_matrix the mixed variants' FP64 diagonal tiles agree
to 5e-14 of max|L| (measured 1.1e-14 at n = 4 096, b = 512) and the backward
error is unchanged to 1e-3 relative (it is set by the SP / HP classes); the
pure-FP64 variant and the exact sp_compute = "fp64" mode never take the INT8
path (bitwise equal)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2408_04440_b200 as sph
n, b, variant, sp, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
h = sph.Cholesky(n, variant, tile_size=b, sp_compute=sp)
h.generate_spd(1)
h.factor()
h.wait()
np.save(out, h.factor_dense())
print(h.residual_probe(1, 2))
''' % ROOT


def _run(tmp_path, n, b, variant, sp, emu):
    f = str(tmp_path / f"L_{variant}_{sp}_{emu}.npy")
    env = dict(os.environ, SPHEMU_DP_EMU=emu)
    r = subprocess.run([sys.executable, "-c", CODE, str(n), str(b), variant, sp, f], env=env, capture_output=True,
                       text=True, timeout=600, check=True)
    return np.load(f), float(r.stdout.split()[-1])


@pytest.mark.parametrize("variant,b", [("dpsp", 512), ("dpsphp", 256), ("dphp", 512)])
def test_int8_dp_update_matches_dmma(tmp_path, variant, b):
    n = 3000
    l0, p0 = _run(tmp_path, n, b, variant, "fp16x3", "0")
    l1, p1 = _run(tmp_path, n, b, variant, "fp16x3", "1")
    scale = np.abs(l0).max()
    for t in range(0, n, b):
        d = np.abs(l0[t:t + b, t:t + b] - l1[t:t + b, t:t + b]).max()
        assert d <= 5e-14 * scale, (t, d / scale)
    assert abs(p1 - p0) <= 1e-3 * p0 + 1e-15, (p0, p1)


@pytest.mark.parametrize("variant,sp", [("dp", "fp16x3"), ("dpsp", "fp64")])
def test_exact_modes_stay_on_dmma(tmp_path, variant, sp):
    l0, _ = _run(tmp_path, 1536, 256, variant, sp, "0")
    l1, _ = _run(tmp_path, 1536, 256, variant, sp, "1")
    assert np.array_equal(l0, l1)
