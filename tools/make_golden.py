"""Writes tests/golden/ref_vectors.npz from oracle/_ref — the reference's own
half.hpp / rng.hpp / wigner.cpp / sht.cpp compiled from /root/reference
(oracle/ref/build_ref.sh). Run here (the reference is not on the GPU box);
the committed fixture then pins the oracle everywhere."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

R = O.ref()
out = {}
b = np.empty(2000)
R.ref_rng_normals(7, 2000, b)
out["rng_normals_seed7"] = b
u = np.empty(1000)
R.ref_rng_uniforms(1, 1000, u)
out["rng_uniforms_seed1"] = u
xs = np.concatenate([[1 / 3, 65505.0, -70000.0, 0.5, 65519.0, 65520.0, 6e-8, 3e-8, -2.98e-8, 1e-300, np.inf, -np.inf],
                     np.random.default_rng(0).standard_normal(4000) * np.logspace(-9, 6, 4000)])
sat = C.c_longlong(0)
out["half_in"] = xs
out["half_out"] = np.array([R.ref_quantize_half(float(x), C.byref(sat)) for x in xs])
out["half_saturations"] = np.array([sat.value])
for L in (13, 33):
    cnt = sum((2 * l + 1) ** 2 for l in range(L))
    d = np.empty(cnt)
    q = np.empty(L * (L + 1) // 2 * L)
    rn = C.c_int()
    R.ref_wigner_dump(L, d, q, C.byref(rn))
    out[f"wigner_d_L{L}"] = d
    out[f"wigner_q_L{L}"] = q
for (nt, nphi, L) in ((9, 16, 8), (33, 64, 16), (17, 20, 9), (46, 90, 45)):
    c = np.stack([O.draw_random_coefficients(L, 100 * L + s) for s in range(2)])
    f = np.empty((2, nt, nphi))
    R.ref_inverse_sht_batch(nt, nphi, L, c, 2, f, 1)
    rng = np.random.default_rng(L)
    x = rng.standard_normal((2, nt, nphi))  # not band-limited: pins the full linear map
    g = np.empty((2, L * L))
    R.ref_forward_sht_batch(nt, nphi, L, x, 2, g, 1)
    out[f"sht_{nt}x{nphi}_L{L}_coeffs"] = c
    out[f"sht_{nt}x{nphi}_L{L}_fields"] = f
    out[f"sht_{nt}x{nphi}_L{L}_x"] = x
    out[f"sht_{nt}x{nphi}_L{L}_fx"] = g
# synth_bandlimited (sht.cpp:435-466) on resolved and under-resolved grids
for (nt, nphi, L) in ((7, 12, 6), (9, 16, 16), (21, 40, 45), (121, 256, 20)):
    c = O.draw_random_coefficients(L, 7 * L + 1)
    f = np.empty((nt, nphi))
    R.ref_synth_bandlimited(c, L, nt, nphi, f)
    out[f"synth_{nt}x{nphi}_L{L}_coeffs"] = c
    out[f"synth_{nt}x{nphi}_L{L}_field"] = f
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "ref_vectors.npz"), **out)
print("wrote", len(out), "arrays")
