"""Emulation from the device-resident tiled factor:
xi = V eta by a TRMM over the stored mixed-precision tiles
(sphemu_gpu_chol_trmm / sphemu_gpu_emulate_chol), against the FP64 product
with the same (quantized) factor and against the dense-V emulate path /
the oracle of stochastic.cpp:217-277.

Tolerances (relative to max|xi|): DP tiles FP64 DMMA 1e-13; SP tiles
fp16 hi/lo x eta hi/lo and HP fp16 tiles x eta's fp16 hi/lo, with fp32
TMEM partial sums over <= max(b, 8192) of K added into FP64: 2e-5 (the
tensor cores' fp32 accumulation truncates: measured 8.9e-6 at K = 8192);
HP bf16 tiles x eta's bf16 hi/lo (16 bits of eta) 1e-4."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {("dp", "fp16"): 1e-13, ("dpsp", "fp16"): 2e-5, ("dpsphp", "fp16"): 2e-5, ("dphp", "fp16"): 2e-5,
       ("dpsphp", "bf16"): 1e-4, ("dphp", "bf16"): 1e-4}


def dense_spd(d, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((2 * d, d))
    a = x.T @ x / (2 * d)
    a[np.diag_indices(d)] += 1e-3
    return 0.5 * (a + a.T)


def factored(sph, a, variant, b, hp="fp16", **kw):
    h = sph.Cholesky(a.shape[0], variant, tile_size=b, hp_format=hp, **kw)
    h.load(a)
    h.factor()
    h.wait()
    return h


@pytest.mark.parametrize("variant,hp", sorted(TOL))
@pytest.mark.parametrize("n,b,S", [(2304, 256, 300), (1900, 256, 257), (3000, 512, 64), (700, 128, 513)])
def test_trmm_matches_fp64_product(sph, variant, hp, n, b, S):
    a = dense_spd(n, 7)
    h = factored(sph, a, variant, b, hp)
    L = h.factor_dense()
    eta = np.random.default_rng(1).standard_normal((S, n))
    got = h.trmm(eta)
    want = eta @ L.T
    err = np.abs(got - want).max() / np.abs(want).max()
    assert err <= TOL[(variant, hp)], err


def test_trmm_band_width_and_fp64_mode(sph):
    """DP tiles off the diagonal (band 2) and the FP64 compute mode's
    64-granule tile pitch (rows of the last 128-row block past the tile)."""
    a = dense_spd(1000, 3)
    for kw in ({"band_width_dp": 2, "sp_fraction": 0.4}, {"compute": "fp64"}):
        h = factored(sph, a, "dpsphp", 200, **kw)
        L = h.factor_dense()
        eta = np.random.default_rng(2).standard_normal((130, 1000))
        got = h.trmm(eta)
        want = eta @ L.T
        assert np.abs(got - want).max() <= 2e-5 * np.abs(want).max()


def test_trmm_needs_a_factor(sph):
    h = sph.Cholesky(300, "dp", tile_size=128)
    with pytest.raises(ValueError, match="no factor"):
        h.trmm(np.zeros((4, 300)))


def _model(L, order, seed=3):
    d = L * L
    rng = np.random.default_rng(seed)
    phi = np.stack([np.full(d, c) for c in (0.5, 0.2, 0.1)[:order]])
    nt, nphi = L + 1, 2 * L
    points = nt * nphi
    return phi, 0.5 + rng.random(points), np.full(points, 0.04), nt, nphi


@pytest.mark.parametrize("rng", ["reference", "philox"])
def test_emulate_chol_matches_dense_v_path(sph, O, rng):
    """The tiled-factor generator equals the dense-V generator (and so the
    oracle, test_gpu_emulate.py) on a dp factor, and stays within the class
    tolerance on a mixed one."""
    Lb, order, t_out, r_len = 32, 3, 12, 3
    d = Lb * Lb
    phi, sigma, v2, nt, nphi = _model(Lb, order)
    means = np.tile(np.linspace(0, 1, nt * nphi), (t_out, 1))
    plan = sph.ShtPlan(nt, nphi, Lb)
    a = dense_spd(d, 5)
    for variant, tol in (("dp", 1e-11), ("dpsphp", 1e-5)):
        h = factored(sph, a, variant, 256)
        v = h.factor_dense()
        got = h.emulate(plan, phi, means, sigma, v2, t_out, seed=9, r_len=r_len, rng=rng)
        want = sph._sphemu.emulate(plan, v, phi, means, sigma, v2, t_out, 9, r_len, rng)
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= tol * np.abs(want).max(), variant
        if variant == "dp" and rng == "reference":
            P = O.Plan(nt, nphi, Lb)
            ref = O.emulate(P, v, phi, means, sigma, v2, t_out, 9, r_len)
            assert np.abs(got - ref).max() < 1e-11 * np.abs(ref).max()


def test_emulate_chol_chunking_is_invisible(sph, tmp_path):
    """Replicate chunks (SPHEMU_EMUL_CHUNK_MB) change nothing: same draws,
    same products, same fields."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import paper_2408_04440_b200 as sph
from test_gpu_emulate_chol import dense_spd, factored, _model
Lb, order, t_out = 24, 2, 10
phi, sigma, v2, nt, nphi = _model(Lb, order)
plan = sph.ShtPlan(nt, nphi, Lb)
h = factored(sph, dense_spd(Lb * Lb, 4), "dpsphp", 128)
out = h.emulate(plan, phi, np.zeros((t_out, nt * nphi)), sigma, v2, t_out, seed=3, r_len=7, rng="philox")
np.save(sys.argv[1], out)
''' % (ROOT, os.path.join(ROOT, "tests"))
    outs = []
    for mb in ("0", "1"):
        f = str(tmp_path / f"e{mb}.npy")
        env = dict(os.environ)
        if mb != "0":
            env["SPHEMU_EMUL_CHUNK_MB"] = mb  # ~1 replicate per chunk
        subprocess.run([sys.executable, "-c", code, f], check=True, env=env, timeout=600)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def test_emulate_chol_replicate_ranges_compose(sph):
    Lb, order, t_out = 16, 2, 8
    phi, sigma, v2, nt, nphi = _model(Lb, order)
    plan = sph.ShtPlan(nt, nphi, Lb)
    h = factored(sph, dense_spd(Lb * Lb, 8), "dpsp", 128)
    means = np.zeros((t_out, nt * nphi))
    full = h.emulate(plan, phi, means, sigma, v2, t_out, seed=5, r_len=5)
    parts = [h.emulate(plan, phi, means, sigma, v2, t_out, seed=5, r_len=c, r_begin=b) for b, c in ((0, 2), (2, 3))]
    assert np.array_equal(np.concatenate(parts), full)
