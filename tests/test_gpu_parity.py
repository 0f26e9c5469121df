"""Parity of the tensor-core path where the flops are:
dense, non-decaying SPD inputs through the b = 256 / 512 tcgen05 path (every
tile O(1), unlike make_spd_test_matrix whose tiles beyond distance 1 vanish),
the strongly correlated KMS generalisation of the reference generator, the
C1-style nugget-regularised covariance, the CTA-pair vs single-CTA HP update,
and the device quantisation known-answer tests (test_mpchol.cpp:177-202).

Stated backward-error bounds (r = ||A - LL^T||_F / ||A||_F, r_ref = the
oracle's on the same input and precision map, u_p = unit roundoff):
  dp                    : elementwise <= 1e-13 relative vs the oracle factor;
  HP classes            : r <= 1.05 r_ref (storage rounding dominates: the
                          fp32-accumulated tensor-core update adds < 1%);
  SP class, fp16x3/tf32x3 (default): r <= 2 r_ref + b 2^-24 — the tensor
                          cores accumulate each tile update's K = b products
                          in truncating fp32, so where the trailing updates
                          cancel (ill-conditioned input) the SP class carries
                          up to ~b ulps of fp32 per step that the FP64 oracle
                          does not;
  SP class, sp_compute="fp64": r <= 1.01 r_ref, elementwise <= 2^-22 (one
                          fp32 rounding flip) — the oracle's arithmetic.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKERS = os.cpu_count() or 8


def dense_spd(d, seed, ratio=2.0, delta=1e-3):
    """A = X^T X / n + delta I with Gaussian X (n = ratio d): kappa ~ 30, O(1) tiles everywhere."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((int(ratio * d), d))
    a = x.T @ x / x.shape[0]
    a = 0.5 * (a + a.T)
    a[np.diag_indices(d)] += delta
    return a


def kms_spd(O, d, seed, rho):
    """make_spd_test_matrix (mpchol.cpp:419-435) with the 0.9 decay replaced by rho:
    D (I + K/4) D with K the Kac-Murdock-Szego matrix, SPD for |rho| < 1."""
    a = O.make_spd(d, seed)
    dd = np.sqrt(np.diag(a) / 1.25)
    i = np.arange(d)
    a = 0.25 * np.outer(dd, dd) * rho ** np.abs(i[:, None] - i[None, :])
    a[i, i] = 1.25 * dd * dd
    return a


_CACHE = {}


def inputs(O, name):
    if name not in _CACHE:
        if name == "xtx2048":
            _CACHE[name] = (dense_spd(2048, 11), 256)
        elif name == "xtx3072":
            _CACHE[name] = (dense_spd(3072, 11), 512)
        elif name == "kms999":
            _CACHE[name] = (kms_spd(O, 3072, 1, 0.999), 512)
        elif name == "kms9999":
            _CACHE[name] = (kms_spd(O, 3072, 1, 0.9999), 512)
    return _CACHE[name]


def run(sph, O, a, variant, b, **kw):
    f, _ = sph.tiled_cholesky(a, variant, tile_size=b, **kw)
    okw = {k: v for k, v in kw.items() if k in ("hp_format",)}
    ref, _ = O.tiled_cholesky(a, variant, tile_size=b, workers=WORKERS, **okw)
    r, r_ref = O.relative_residual(a, f), O.relative_residual(a, ref)
    elem = np.abs(f - ref).max() / np.abs(ref).max()
    return r, r_ref, elem


INPUTS = ["xtx2048", "xtx3072", "kms999", "kms9999"]


@pytest.mark.parametrize("name", INPUTS)
def test_dp_factor_elementwise(sph, O, name):
    a, b = inputs(O, name)
    r, r_ref, elem = run(sph, O, a, "dp", b)
    assert elem <= 1e-13 and r <= 2 * r_ref + 1e-15, (elem, r, r_ref)


@pytest.mark.parametrize("name", INPUTS)
@pytest.mark.parametrize("variant,hp", [("dpsphp", "fp16"), ("dpsphp", "bf16"), ("dphp", "fp16"), ("dphp", "bf16")])
def test_hp_classes_match_oracle(sph, O, name, variant, hp):
    a, b = inputs(O, name)
    r, r_ref, elem = run(sph, O, a, variant, b, hp_format=hp)
    assert r <= 1.05 * r_ref, (r, r_ref)
    # one storage rounding of a few entries differs (2^-11 fp16, 2^-8 bf16, times the factor's scale)
    assert elem <= (8 * 2.0 ** -11 if hp == "fp16" else 8 * 2.0 ** -8), elem


@pytest.mark.parametrize("name", INPUTS)
@pytest.mark.parametrize("spc", ["fp16x3", "tf32x3"])
def test_sp_class_tensor_bound(sph, O, name, spc):
    a, b = inputs(O, name)
    r, r_ref, elem = run(sph, O, a, "dpsp", b, sp_compute=spc)
    assert r <= 2 * r_ref + b * 2.0 ** -24, (r, r_ref)
    assert elem <= b * 2.0 ** -24, elem
    if name.startswith("xtx"):
        assert r <= 5e-6  # the reference threshold (acceptance_main.cpp:226) on well-conditioned input


@pytest.mark.parametrize("name", INPUTS)
@pytest.mark.parametrize("variant", ["dpsp", "dpsphp"])
def test_sp_fp64_mode_is_the_oracle(sph, O, name, variant):
    a, b = inputs(O, name)
    r, r_ref, elem = run(sph, O, a, variant, b, sp_compute="fp64")
    assert r <= 1.01 * r_ref, (r, r_ref)
    if variant == "dpsp":
        assert elem <= 2.0 ** -22, elem


def test_cta_pair_and_single_cta_hp_update_are_bitwise_equal(O, tmp_path):
    """The HP update's CTA-pair form (cta_group::2, M = 256, 16-warp epilogue,
    the default at b % 256 == 0) and its single-CTA form must agree bitwise on
    dense input (SPHEMU_TC_CG is read once per process: one subprocess each)."""
    a = dense_spd(3072, 5)
    path = str(tmp_path / "cg_in.npy")
    np.save(path, a)
    outs = []
    for cg in ("2", "1"):
        out = path.replace("cg_in", f"cg_out{cg}")
        code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_2408_04440_b200 as s; "
                "a = np.load(%r); f, _ = s.tiled_cholesky(a, 'dphp', tile_size=512, hp_format='bf16'); "
                "g, _ = s.tiled_cholesky(a, 'dpsphp', tile_size=256, hp_format='fp16', sp_fraction=0.3); "
                "np.save(%r, np.stack([f[:3072, :3072], g]))" % (ROOT, path, out))
        env = dict(os.environ, SPHEMU_TC_CG=cg)
        subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
    ref, _ = O.tiled_cholesky(a, "dphp", tile_size=512, hp_format="bf16", workers=WORKERS)
    assert O.relative_residual(a, outs[0][0]) <= 1.05 * O.relative_residual(a, ref)


# ---- C1-style covariance: n = 97 < d = 2025, nugget-regularised ----------
def c1_residuals(rank, seed=91):
    rng = np.random.default_rng(seed)
    d, n = 2025, 97
    basis = rng.standard_normal((rank, d)) / (1.0 + np.arange(d) % 45) ** 0.5
    return rng.standard_normal((n, rank)) @ basis


def oracle_cov(O, xi, variant, tile):
    import ctypes as C
    n, d = xi.shape
    u, v = np.empty((d, d)), np.empty((d, d))
    nug = C.c_double()
    st = O.CholStats()
    cfg = O.config(variant, tile)
    rc = O.lib().so_estimate_innovation_covariance(np.ascontiguousarray(xi), n, d, C.byref(cfg), 1, u, v,
                                                   C.byref(nug), C.byref(st))
    return rc, u, v, nug.value


@pytest.mark.parametrize("rank", [97, 40])
@pytest.mark.parametrize("variant,b", [("dp", 256), ("dp", 512), ("dpsp", 256), ("dpsp", 512), ("dpsphp", 512)])
def test_c1_nugget_covariance_vs_oracle(sph, O, rank, variant, b):
    """estimate_innovation_covariance (stochastic.cpp:109-172) with a mixed
    precision map through the b = 256/512 path: the SP class in its FP64
    mode (the default of this entry point) picks the oracle's nugget and
    reaches the oracle's backward error."""
    xi = c1_residuals(rank)
    n = xi.shape[0]
    rc, uo, vo, nugo = oracle_cov(O, xi, variant, b)
    try:
        u, v, nug, _ = sph._sphemu.estimate_innovation_covariance(xi, 1, n + 3, 3, variant=variant, tile_size=b)
    except RuntimeError:
        assert rc != 0  # the oracle gives up too
        return
    assert rc == 0
    assert np.abs(u - uo).max() <= 1e-12 * np.abs(uo).max()
    assert nug == nugo, (nug, nugo)
    r = O.relative_residual(u + nug * np.eye(u.shape[0]), v)
    r_ref = O.relative_residual(uo + nugo * np.eye(u.shape[0]), vo)
    # HP: storage rounding dominates, the order of the fp32 tensor-core sums shifts it by up to ~10 %
    assert r <= (2 if variant == "dp" else 1.15 if variant == "dpsphp" else 1.01) * r_ref + 1e-15, (r, r_ref)


def test_c1_nugget_covariance_fp16x3_escalates_no_lower(sph, O):
    """With the fast SP arithmetic the nugget loop may need a larger nugget
    than the oracle (never a smaller one), and the factor it returns still
    meets the SP bound."""
    xi = c1_residuals(97)
    n = xi.shape[0]
    rc, uo, vo, nugo = oracle_cov(O, xi, "dpsp", 256)
    u, v, nug, _ = sph._sphemu.estimate_innovation_covariance(xi, 1, n + 3, 3, variant="dpsp", tile_size=256,
                                                               sp_compute="fp16x3")
    assert rc == 0 and nug >= nugo
    assert O.relative_residual(u + nug * np.eye(u.shape[0]), v) <= 5e-6


# ---- device quantisation KATs (test_mpchol.cpp:177-202; half.hpp) ---------
def _kat_matrix(vals, n=128, b=32):
    a = np.zeros((n, n))
    a[np.diag_indices(n)] = 1e6
    rows, cols = np.tril_indices(n, -b)  # strictly below the DP band: the HP tiles of dphp
    sel = [(r, c) for r, c in zip(rows, cols) if r // b - c // b >= 1][: len(vals)]
    for (r, c), x in zip(sel, vals):
        a[r, c] = x
        a[c, r] = x
    return a, sel


@pytest.mark.parametrize("compute", ["tensor", "fp64"])
def test_device_half_quantization_kat(sph, O, G, compute):
    """The reference's binary16 golden vectors (tests/golden: half_in -> half_out
    and the saturation count, generated from half.hpp itself) pushed through
    the device load path (chol_load_dense -> HP tiles -> store_dense)."""
    vals = G["half_in"]
    a, sel = _kat_matrix(vals)
    h = sph.Cholesky(a.shape[0], "dphp", tile_size=32, compute=compute)
    h.load(a)
    st = h.wait()
    f = h.factor_dense_unfactored()
    got = np.array([f[r, c] for r, c in sel])
    assert np.array_equal(got, G["half_out"][: len(sel)])
    assert st.half_saturations == int(G["half_saturations"][0])


def test_device_quantization_kats_single_and_bf16(sph, O):
    """test_mpchol.cpp:177-202 KATs on the device: 1/3 -> float exactly (SP),
    0.333251953125 (HP), 65505 -> 65504 not counted, -70000 -> -65504 counted;
    the bf16 class against the oracle's bf16 quantizer."""
    n, b = 128, 32
    a = np.zeros((n, n))
    a[np.diag_indices(n)] = 1e6
    a[40, 0] = a[0, 40] = 1.0 / 3.0
    a[41, 1] = a[1, 41] = 65505.0
    a[42, 2] = a[2, 42] = -70000.0
    h = sph.Cholesky(n, "dpsphp", tile_size=b, sp_fraction=1.0)  # all off-band tiles SP
    h.load(a)
    h.wait()
    f = h.factor_dense_unfactored()
    assert f[40, 0] == float(np.float32(1.0 / 3.0))
    h = sph.Cholesky(n, "dphp", tile_size=b)
    h.load(a)
    st = h.wait()
    f = h.factor_dense_unfactored()
    assert f[40, 0] == 0.333251953125 and f[41, 1] == 65504.0 and f[42, 2] == -65504.0
    assert st.half_saturations == 1
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.integers(-40, 40, 2000), [3.4e38, -3.5e38, 1e-45]])
    a, sel = _kat_matrix(vals, n=256)
    h = sph.Cholesky(256, "dphp", tile_size=32, hp_format="bf16")
    h.load(a)
    h.wait()
    f = h.factor_dense_unfactored()
    got = np.array([f[r, c] for r, c in sel])
    want, _ = O.quantize(np.array(vals[: len(sel)]), 2, hp_format="bf16")
    assert np.array_equal(got, want)


def test_epilogue_saturation_matches_oracle(sph, O):
    """A trailing update that overflows binary16 inside the tcgen05 epilogue
    (cvt.rn.satfinite) saturates and is counted exactly like quantize_tile."""
    b, n = 256, 768
    s, t = 300.0, 250.0  # L10 = s I, L20 = t I  ->  update of tile (2,1) = -s t I = -75000 I
    a = np.zeros((n, n))
    i = np.arange(b)
    a[i, i] = 1.0
    a[b + i, i] = a[i, b + i] = s
    a[2 * b + i, i] = a[i, 2 * b + i] = t
    a[b + i, b + i] = s * s + 1e6
    a[2 * b + i, 2 * b + i] = t * t + 1e12
    for compute in ("tensor", "fp64"):
        f, js = sph.tiled_cholesky(a, "dphp", tile_size=b, compute=compute)
        ref, ro = O.tiled_cholesky(a, "dphp", tile_size=b)
        import json
        assert json.loads(js)["conversions"]["half_saturations"] == ro["conversions"]["half_saturations"] > 0
        assert np.abs(f - ref).max() <= 1e-3 * np.abs(ref).max()


# ---- tile-norm precision policy (opt-in next to mpchol.cpp:67-93) ----
@pytest.mark.parametrize("name", ["xtx2048", "kms999"])
@pytest.mark.parametrize("variant", ["dpsp", "dpsphp", "dphp"])
def test_tile_norm_policy_matches_oracle(sph, O, name, variant):
    """The device tile norms give the oracle's map; the factorization on that
    map matches the oracle run on the same map within the class bounds, and
    the backward error stays at the policy's tolerance scale."""
    a, b = inputs(O, name)
    for tol in (1e-6, 1e-9):
        pm = sph.tile_norm_precisions(a, variant, b, tolerance=tol)
        assert np.array_equal(pm, O.tile_norm_precisions(a, variant, b, tolerance=tol))
        f, js = sph.tiled_cholesky(a, variant, tile_size=b, precision_policy="norm", norm_tolerance=tol,
                                   sp_compute="fp64")
        ref, st = O.tiled_cholesky(a, variant, tile_size=b, workers=WORKERS, precision_map=pm)
        r, r_ref = O.relative_residual(a, f), O.relative_residual(a, ref)
        assert r <= 1.15 * r_ref + 1e-15, (tol, r, r_ref)


def test_tile_norm_policy_on_reference_generator(sph, O):
    """On make_spd_test_matrix the norm rule demotes the vanishing far tiles to
    HP and keeps the distance-1 tiles wide: far better accuracy than the band
    rule's dpsphp at nearly the same memory."""
    a = O.make_spd(2048, 1)
    pm = sph.tile_norm_precisions(a, "dpsphp", 256, tolerance=1e-8)
    nt = 8
    dist1 = [pm[i * (i + 1) // 2 + i - 1] for i in range(1, nt)]
    far = [pm[i * (i + 1) // 2 + j] for i in range(nt) for j in range(i - 1)]
    assert all(p != 2 for p in dist1) and all(p == 2 for p in far)
    f, _ = sph.tiled_cholesky(a, "dpsphp", tile_size=256, precision_policy="norm", norm_tolerance=1e-8)
    g, _ = sph.tiled_cholesky(a, "dpsphp", tile_size=256)
    assert O.relative_residual(a, f) < 1e-6 < O.relative_residual(a, g)
