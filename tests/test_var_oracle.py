"""CPU: the numpy restatement of fit_var (stochastic.cpp:30-107) against the
reference's own fit_var tests (test_stochastic.cpp:93-157). The reference
needs Eigen (absent), so these known answers pin the restatement."""
import numpy as np


def ar2_series(r_len, t_len, phi1, phi2, scale, seed):
    rng = np.random.default_rng(seed)
    d = phi1.size
    c = np.zeros((r_len, t_len, d))
    for r in range(r_len):
        for t in range(t_len):
            e = scale * rng.standard_normal(d)
            c[r, t] = e + (phi1 * c[r, t - 1] if t >= 1 else 0) + (phi2 * c[r, t - 2] if t >= 2 else 0)
    return c


def test_lag_coefficients_recovered(O):  # test_stochastic.cpp:93-123
    i = np.arange(9.0)
    phi1, phi2, scale = 0.45 + 0.03 * i, -0.25 + 0.02 * i, 0.5 + 0.1 * i
    fit = O.fit_var(ar2_series(2, 3000, phi1, phi2, scale, 424242), 2)
    assert fit["zeroed_count"] == 0 and fit["unstable_count"] == 0
    assert fit["residuals"].shape == (2 * 2998, 9)
    assert fit["residual_mean_norm"] < 0.05
    assert np.all(fit["phi_se"] > 0)
    err = np.abs(fit["phi"] - np.stack([phi1, phi2]))
    assert np.all(err < 4 * fit["phi_se"]) and np.sum(err >= 3 * fit["phi_se"]) <= 1


def test_order_zero_demeans(O):  # test_stochastic.cpp:125-142
    c = np.random.default_rng(5).standard_normal((2, 6, 4))
    fit = O.fit_var(c, 0)
    assert fit["phi"].shape == (0, 4) and fit["residuals"].shape == (12, 4)
    assert np.allclose(fit["residuals"], (c - c.reshape(-1, 4).mean(axis=0)).reshape(12, 4), rtol=1e-14, atol=1e-15)


def test_silent_and_explosive_flagged(O):  # test_stochastic.cpp:144-157
    c = np.zeros((1, 400, 4))
    c[0, :, 0] = np.arange(1, 401, dtype=np.float64)
    fit = O.fit_var(c, 1)
    assert fit["zeroed_count"] == 3 and fit["unstable_count"] == 1
    assert fit["phi"][0, 0] > 1.0 and np.all(fit["phi"][0, 1:] == 0.0)
