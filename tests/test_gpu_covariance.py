"""GPU innovation covariance + nugget loop (stochastic.cpp:109-172) against
the oracle restatement, with the reference's own checks
(test_stochastic.cpp:159-210: U = Xi^T Xi / n to 1e-12, V V^T = U + nugget I
to 1e-12, nugget escalation)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def oracle_cov(O, xi, variant, tile):
    n, d = xi.shape
    u = np.empty((d, d))
    v = np.empty((d, d))
    nug = C.c_double()
    st = O.CholStats()
    cfg = O.config(variant, tile)
    rc = O.lib().so_estimate_innovation_covariance(np.ascontiguousarray(xi), n, d, C.byref(cfg), 1, u, v,
                                                   C.byref(nug), C.byref(st))
    return rc, u, v, nug.value


def residuals(n, d, seed, rank=None):
    rng = np.random.default_rng(seed)
    if rank is None:
        return rng.standard_normal((n, d)) * (1.0 / (1.0 + np.arange(d) % 7))
    basis = rng.standard_normal((rank, d))
    return rng.standard_normal((n, rank)) @ basis


@pytest.mark.parametrize("r_len,t_len,order,d,tile,variant", [
    (2, 50, 2, 64, 32, "dp"),      # n = 96 > d: no nugget
    (1, 40, 3, 64, 32, "dp"),      # n = 37 < d: nugget from 1e-8 mean(diag)
    (3, 200, 1, 100, 32, "dpsp"),  # ragged tiles, mixed precision
    (4, 130, 2, 256, 64, "dp"),
])
def test_covariance_matches_oracle(sph, O, r_len, t_len, order, d, tile, variant):
    n = r_len * (t_len - order)
    xi = residuals(n, d, seed=7 + d)
    u, v, nug, stats = sph._sphemu.estimate_innovation_covariance(xi, r_len, t_len, order, variant=variant,
                                                                   tile_size=tile)
    rc, uo, vo, nugo = oracle_cov(O, xi, variant, tile)
    assert rc == 0
    want_u = xi.T @ xi / n
    assert np.abs(u - u.T).max() == 0.0  # exactly symmetric like the reference's (U + U^T) / 2
    assert np.abs(u - want_u).max() <= 1e-12 * np.abs(want_u).max()
    assert np.abs(u - uo).max() <= 1e-12 * np.abs(uo).max()
    assert nug == nugo
    assert np.abs(np.triu(v, 1)).max() == 0.0
    target = u + nug * np.eye(d)
    tol = 1e-12 if variant == "dp" else 5e-6
    assert np.abs(v @ v.T - target).max() <= tol * np.abs(target).max()
    if variant == "dp":
        assert np.abs(v - vo).max() <= 1e-10 * np.abs(vo).max()


def test_rank_deficient_escalates_like_oracle(sph, O):
    # rank 5 innovations in d = 64: singular U, the nugget must be raised
    r_len, t_len, order, d = 2, 30, 1, 64
    n = r_len * (t_len - order)
    xi = residuals(n, d, seed=3, rank=5)
    u, v, nug, _ = sph._sphemu.estimate_innovation_covariance(xi, r_len, t_len, order, tile_size=32)
    rc, uo, vo, nugo = oracle_cov(O, xi, "dp", 32)
    assert rc == 0 and nug == nugo and nug > 0.0
    assert np.abs(v @ v.T - (u + nug * np.eye(d))).max() <= 1e-12 * np.abs(u).max()


def test_shape_errors(sph):
    xi = np.ones((10, 4))
    with pytest.raises(ValueError, match="row count"):
        sph._sphemu.estimate_innovation_covariance(xi, 2, 10, 1)  # 2 * 9 != 10
    with pytest.raises(ValueError, match="too small"):
        sph._sphemu.estimate_innovation_covariance(np.ones((1, 4)), 1, 2, 1)
    with pytest.raises(RuntimeError, match="mean diagonal"):
        sph._sphemu.estimate_innovation_covariance(np.zeros((10, 4)), 1, 11, 1)
