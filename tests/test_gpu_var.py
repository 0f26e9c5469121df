"""GPU fit_var (var.cu) against the numpy restatement of stochastic.cpp:30-107
and the reference's fit_var tests; the residuals feed the device covariance."""
import numpy as np
import pytest

from test_var_oracle import ar2_series

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order", [0, 1, 2, 3])
def test_fit_var_matches_oracle(sph, O, order):
    i = np.arange(36.0)
    c = ar2_series(3, 200, 0.4 + 0.005 * i, -0.2 + 0.004 * i, 0.5 + 0.01 * i, 7)
    got = sph.fit_var(c, order)
    want = O.fit_var(c, order)
    tol = 1e-12
    assert np.abs(got.phi - want["phi"]).max(initial=0) < tol
    assert np.abs(got.phi_se - want["phi_se"]).max(initial=0) < tol * max(1.0, np.abs(want["phi_se"]).max(initial=0))
    assert np.abs(got.residuals - want["residuals"]).max() < tol * np.abs(c).max()
    assert got.zeroed_count == want["zeroed_count"] and got.unstable_count == want["unstable_count"]
    assert abs(got.residual_mean_norm - want["residual_mean_norm"]) < 1e-12


def test_lag_coefficients_recovered(sph):  # test_stochastic.cpp:93-123
    i = np.arange(9.0)
    phi1, phi2, scale = 0.45 + 0.03 * i, -0.25 + 0.02 * i, 0.5 + 0.1 * i
    fit = sph.fit_var(ar2_series(2, 3000, phi1, phi2, scale, 424242), 2)
    assert fit.zeroed_count == 0 and fit.unstable_count == 0 and fit.residual_mean_norm < 0.05
    err = np.abs(fit.phi - np.stack([phi1, phi2]))
    assert np.all(err < 4 * fit.phi_se) and np.sum(err >= 3 * fit.phi_se) <= 1


def test_silent_and_explosive_flagged(sph):  # test_stochastic.cpp:144-157
    c = np.zeros((1, 400, 4))
    c[0, :, 0] = np.arange(1, 401, dtype=np.float64)
    fit = sph.fit_var(c, 1)
    assert fit.zeroed_count == 3 and fit.unstable_count == 1
    assert fit.phi[0, 0] > 1.0 and np.all(fit.phi[0, 1:] == 0.0) and np.all(np.isfinite(fit.phi))


def test_unstable_matches_companion_eigenvalues(sph, O):
    # Random AR(3) lag polynomials around the stability boundary: the device's
    # Schur-Cohn decision equals the reference's eigenvalue test.
    rng = np.random.default_rng(3)
    c = rng.standard_normal((2, 60, 512)) * 0.1
    c[:, :, :256] = np.cumsum(c[:, :, :256], axis=1)  # random walks: roots near 1
    got = sph.fit_var(c, 3)
    want = O.fit_var(c, 3)
    assert got.unstable_count == want["unstable_count"]


def test_errors_and_feeds_covariance(sph):
    with pytest.raises(ValueError):
        sph.fit_var(np.zeros((1, 2, 4)), 2)
    with pytest.raises(ValueError):
        sph.fit_var(np.zeros((1, 5, 4)), -1)
    i = np.arange(16.0)
    c = ar2_series(2, 300, 0.3 + 0 * i, -0.1 + 0 * i, 1.0 + 0 * i, 11)
    fit = sph.fit_var(c, 2)
    u, v, nug, _ = sph.estimate_innovation_covariance(fit.residuals, 2, 300, 2, tile_size=8)
    assert np.abs(u - fit.residuals.T @ fit.residuals / fit.residuals.shape[0]).max() < 1e-12
