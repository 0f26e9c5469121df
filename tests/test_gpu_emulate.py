"""GPU emulation generator vs the oracle restatement of stochastic.cpp:217-277
(reference RNG stream, so the draws are identical up to GEMV summation order)
and a statistics screen for the device Philox stream."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def model(O, L, order, seed=3):
    d = L * L
    rng = np.random.default_rng(seed)
    u = np.array([[0.3 * 0.7 ** abs(i - j) for j in range(d)] for i in range(d)])
    v = O.dense_cholesky(u)
    phi = np.stack([np.full(d, c) for c in (0.5, 0.2, 0.1)[:order]]) if order else np.zeros((0, d))
    nt, nphi = L + 1, 2 * L
    points = nt * nphi
    sigma = 0.5 + rng.random(points)
    v2 = np.full(points, 0.04)
    return v, phi, sigma, v2, nt, nphi


def run_gpu(sph, L, nt, nphi, v, phi, means, sigma, v2, t_out, seed, r_len, rng_mode):
    plan = sph.ShtPlan(nt, nphi, L)
    return sph._sphemu.emulate(plan, v, phi if phi.shape[0] else None, means, sigma, v2, t_out, seed, r_len,
                               ["reference", "philox"][rng_mode])


@pytest.mark.parametrize("L,order", [(4, 1), (6, 3), (8, 2)])
def test_reference_stream_matches_oracle(sph, O, L, order):
    v, phi, sigma, v2, nt, nphi = model(O, L, order)
    t_out, r_len = 24, 3
    means = np.tile(np.linspace(0, 1, nt * nphi), (t_out, 1)) + np.arange(t_out)[:, None] * 0.01
    got = run_gpu(sph, L, nt, nphi, v, phi, means, sigma, v2, t_out, 11, r_len, 0)
    P = O.Plan(nt, nphi, L)
    want = O.emulate(P, v, phi if order else None, means, sigma, v2, t_out, 11, r_len)
    assert np.abs(got - want).max() < 1e-11 * np.abs(want).max()


def test_philox_stream_statistics(sph, O):
    L = 4
    v, phi, sigma, v2, nt, nphi = model(O, L, 1)
    t_out, r_len = 2000, 4
    means = np.zeros((t_out, nt * nphi))
    a = run_gpu(sph, L, nt, nphi, v, phi, means, sigma, v2, t_out, 5, r_len, 1)
    b = run_gpu(sph, L, nt, nphi, v, phi, means, sigma, v2, t_out, 5, r_len, 0)
    # same model, different streams: per-location variances agree within 10%
    va, vb = a.reshape(-1, nt * nphi).var(0), b.reshape(-1, nt * nphi).var(0)
    assert np.abs(va / vb - 1).max() < 0.1
    assert np.abs(a.mean(axis=(0, 1))).max() < 5 * np.sqrt(va.max() / (t_out * r_len) * 10)


@pytest.mark.parametrize("rng_mode", [0, 1])
def test_replicate_ranges_compose(sph, O, rng_mode):
    """replicate ranges run independently (one GPU each, no
    communication) and reproduce the single call bitwise."""
    L, order = 6, 2
    v, phi, sigma, v2, nt, nphi = model(O, L, order)
    t_out, r_len = 12, 5
    means = np.zeros((t_out, nt * nphi))
    plan = sph.ShtPlan(nt, nphi, L)
    mode = ["reference", "philox"][rng_mode]
    full = sph._sphemu.emulate(plan, v, phi, means, sigma, v2, t_out, 21, r_len, mode)
    parts = [sph._sphemu.emulate(plan, v, phi, means, sigma, v2, t_out, 21, cnt, mode, r_begin=beg)
             for beg, cnt in ((0, 2), (2, 1), (3, 2))]
    assert np.array_equal(np.concatenate(parts), full)


def _ar_psi_weights(phi):  # tests/support/reference.cpp:123-133
    psi = [1.0]
    for s in range(1, 100000):
        v = sum(phi[j - 1] * psi[s - j] for j in range(1, min(len(phi), s) + 1))
        if s > len(phi) and abs(v) < 1e-12:
            break
        psi.append(v)
    return np.array(psi)


def test_acceptance8_emulation_consistency(sph):
    """acceptance_main.cpp:383-531 (criterion 8): L = 8 on the 9 x 16 grid,
    dense innovation covariance U_ij = d_i d_j 0.7^|i-j|, AR(3) by degree
    (make_generating_model(0.25, 0.75, 0.8), :249-300), v^2 = 0.04, 200
    replicates x 48 steps, seed 88. Screens as the reference: per-location
    3-SE mean and variance screens (<= 2 of 144 locations each, variance
    against the model-implied value) and the hp/dp std ratio (< 0.10) with
    the factor of the same covariance stored in half precision (dphp). The
    factors are the device's; the draws follow the reference stream."""
    L, d, t_len, reps = 8, 64, 48, 200
    nt, nphi = L + 1, 2 * L
    points = nt * nphi
    deg = np.sqrt(np.arange(d)).astype(int)
    di = 0.3 * (1.0 + 0.2 * np.sin(0.37 * np.arange(d)))
    u = di[:, None] * di[None, :] * 0.7 ** np.abs(np.arange(d)[:, None] - np.arange(d)[None, :])
    g = 0.25 + (0.75 - 0.25) * np.arange(L) / (L - 1)
    phi_deg = np.stack([0.60 * g, 0.25 * g, 0.15 * g])
    phi = phi_deg[:, deg]
    sigma = 0.5 + 1.5 * ((7 * np.arange(points)) % 144) / 143.0
    v2 = np.full(points, 0.04)
    tt = np.arange(1, t_len + 1)[:, None]
    means = 0.8 + 0.5 * np.cos(2 * np.pi * tt / 12) - 0.3 * np.sin(2 * np.pi * tt / 12) + np.zeros((1, points))
    plan = sph.ShtPlan(nt, nphi, L)
    f_dp, _ = sph.tiled_cholesky(u, variant="dp", tile_size=16)
    f_hp, _ = sph.tiled_cholesky(u, variant="dphp", tile_size=16)
    y = sph._sphemu.emulate(plan, f_dp, phi, means, sigma, v2, t_len, 88, reps, "reference").reshape(reps, t_len, -1)
    y_hp = sph._sphemu.emulate(plan, f_hp, phi, means, sigma, v2, t_len, 88, reps, "reference").reshape(reps, t_len, -1)
    # model-implied per-location variance (:416-456)
    psi = [_ar_psi_weights(phi_deg[:, l]) for l in range(L)]
    s_ll = np.array([[np.dot(psi[a][:min(len(psi[a]), len(psi[b]))], psi[b][:min(len(psi[a]), len(psi[b]))])
                      for b in range(L)] for a in range(L)])
    cols = plan.inverse(np.eye(d)).reshape(d, points)
    w = u * s_ll[deg][:, deg]
    implied = sigma ** 2 * (np.einsum("il,ij,jl->l", cols, w, cols) + 0.04)
    dev = y - means[None]
    a_rep, b_rep = dev.mean(1), (dev ** 2).mean(1)
    z_mean = a_rep.mean(0) / np.sqrt(a_rep.var(0, ddof=1) / reps)
    z_std = (b_rep.mean(0) - implied) / np.sqrt(b_rep.var(0, ddof=1) / reps)
    ratio = np.sqrt(((y_hp - means[None]) ** 2).sum((0, 1)) / (dev ** 2).sum((0, 1)))
    assert (np.abs(z_mean) > 3).sum() <= 2, np.abs(z_mean).max()
    assert (np.abs(z_std) > 3).sum() <= 2, np.abs(z_std).max()
    assert np.abs(ratio - 1).max() < 0.10


@pytest.mark.parametrize("forcing", [None, (np.linspace(0.2, 1.0, 4), np.array([0.1, 0.05]))])
def test_trend_model_overload(sph, O, forcing):
    """emulate with the TrendModel records (stochastic.cpp:229 mean_table on
    the device) equals emulate with the oracle's mean table and sigma column,
    bitwise (same draws, same device arithmetic)."""
    L, order, K, period, t_out, r_len, t_start = 6, 2, 2, 12, 24, 2, 5
    v, phi, _, v2, nt, nphi = model(O, L, order)
    rng = np.random.default_rng(4)
    rec = rng.standard_normal((nt * nphi, 5 + 2 * K))
    rec[:, 2] = 0.3
    rec[:, 3] = 0.6
    rec[:, -1] = 0.5 + rng.random(nt * nphi)
    means = O.mean_table(rec, K, period, t_out, t_start, forcing=forcing)
    plan = sph.ShtPlan(nt, nphi, L)
    want = sph._sphemu.emulate(plan, v, phi, means, rec[:, -1].copy(), v2, t_out, 13, r_len)
    got = sph.emulate_model(plan, v, phi, rec, K, period, v2, t_out, 13, r_len, t_start=t_start, forcing=forcing)
    assert np.array_equal(got, want)
    with pytest.raises(ValueError):
        sph.emulate_model(plan, v, phi, rec, K, period, v2, t_out, 13, r_len, t_start=0)
