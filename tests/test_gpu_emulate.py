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
