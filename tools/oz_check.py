"""DP-class update on INT8 tensor cores (SPHEMU_DP_EMU=1, default) vs FP64
DMMA (SPHEMU_DP_EMU=0): factor the same matrices both ways and compare the
factors and the backward errors (tools/oz_check.py [N] [B])."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
b = int(sys.argv[2]) if len(sys.argv) > 2 else 512

CODE = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2408_04440_b200 as sph
n, b, variant, kind, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
if kind == "gen":
    h = sph.Cholesky(n, variant, tile_size=b)
    h.generate_spd(1)
    h.factor(); h.wait()
    np.save(out, h.factor_dense())
    print("probe", h.residual_probe(1, 2))
else:
    rng = np.random.default_rng(5)
    x = rng.standard_normal((n + 64, n))
    a = x.T @ x / (n + 64)
    a[np.diag_indices(n)] += 1e-3
    h = sph.Cholesky(n, variant, tile_size=b)
    h.load(0.5 * (a + a.T)); h.factor(); h.wait()
    np.save(out, h.factor_dense())
''' % ROOT

for variant in ("dp", "dpsp", "dpsphp"):
    for kind in ("gen", "dense"):
        fs = []
        for emu in ("0", "1"):
            f = f"/tmp/oz_{variant}_{kind}_{emu}.npy"
            env = dict(os.environ, SPHEMU_DP_EMU=emu)
            r = subprocess.run([sys.executable, "-c", CODE, str(n), str(b), variant, kind, f], env=env,
                               capture_output=True, text=True, timeout=900)
            if r.returncode:
                print(r.stderr[-2000:])
                sys.exit(1)
            fs.append(np.load(f))
            if r.stdout.strip():
                print(variant, kind, "emu", emu, r.stdout.strip())
        d = np.abs(fs[0] - fs[1]).max()
        scale = np.abs(fs[0]).max()
        # diagonal tiles only (the DP class under band 1)
        dd = 0.0
        for t in range(0, n, b):
            dd = max(dd, np.abs(fs[0][t:t + b, t:t + b] - fs[1][t:t + b, t:t + b]).max())
        print(f"{variant:7s} {kind:5s}: max|L_emu - L_dmma| = {d:.3e} (rel {d / scale:.3e}), diagonal tiles {dd / scale:.3e}")
