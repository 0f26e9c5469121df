"""CPU: the oracle restatement of the trend mean structure (trend.cpp:18-83,
252-324) against the reference's own trend tests (test_trend.cpp) and closed
forms. The reference's trend.cpp needs Eigen (fit_trend), so it cannot be
compiled into oracle/_ref here; these known answers pin the restatement."""
import math

import numpy as np
import pytest


def records(points, k, seed=1, lag=0.0):
    rng = np.random.default_rng(seed)
    rec = rng.standard_normal((points, 5 + 2 * k))
    rec[:, 2] = lag
    rec[:, 3] = 0.6
    rec[:, -1] = 0.5 + rng.random(points)
    return rec


def test_mean_table_matches_pointwise(O):  # test_trend.cpp:195-206 (t_start 13, 24 steps, K=1, period 12)
    rec = records(12, 1)
    t = O.mean_table(rec, 1, 12, 24, 13)
    for row in range(24):
        for loc in range(12):
            assert t[row, loc] == O.eval_mean_trend(rec, 1, 12, loc, 13 + row)


def test_closed_form_harmonics(O):
    # t % period == 0 -> base = 0: m = beta0 + sum_k a_k (cos 0 = 1, sin 0 = 0).
    rec = records(5, 3)
    t = O.mean_table(rec, 3, 12, 1, 12)
    assert np.array_equal(t[0], rec[:, 0] + rec[:, 4] + rec[:, 5] + rec[:, 6])
    # quarter period: base = pi/2, k = 1 -> sin = 1.
    rec1 = records(4, 1)
    t = O.mean_table(rec1, 1, 12, 1, 3)
    want = rec1[:, 0] + (rec1[:, 4] * math.cos(math.pi / 2) + rec1[:, 5] * 1.0)
    assert np.allclose(t[0], want, rtol=0, atol=1e-15)


def test_forcing_terms(O):
    # x = year k+1, history[0] = year 0; lagged mean (1-rho) sum rho^{s-1} x_{year-s}.
    rec = records(3, 0, lag=0.5)
    x = np.array([1.0, 2.0, 4.0])
    hist = np.array([0.5, 0.25])
    t = O.mean_table(rec, 0, 12, 36, 1, forcing=(x, hist))
    rho = 0.6
    for year in (1, 2, 3):
        lag = 0.0
        w = 1.0
        for s in range(1, 10):
            y = year - s
            if y >= 1:
                v = x[y - 1]
            elif -y < hist.size:
                v = hist[-y]
            else:
                break
            lag += w * v
            w *= rho
        lag *= 1 - rho
        row = (year - 1) * 12
        want = rec[:, 0] + (rec[:, 1] * x[year - 1] + rec[:, 2] * lag)
        assert np.array_equal(t[row], want)


def test_missing_lag_history_fails(O):  # test_trend.cpp:208-224
    rec = records(3, 0, lag=0.5)
    with pytest.raises(ValueError):
        O.mean_table(rec, 0, 12, 12, 1, forcing=(np.array([1.0]), None))
    # No lag coefficient: the same trajectory evaluates.
    O.mean_table(records(3, 0, lag=0.0), 0, 12, 12, 1, forcing=(np.array([1.0]), None))


def test_time_steps_one_based(O):
    with pytest.raises(ValueError):
        O.mean_table(records(2, 1), 1, 12, 4, 0)


def test_detrend_retrend_identity(O):  # test_trend.cpp:165-193
    rec = records(12, 2, seed=31)
    y = np.random.default_rng(5).standard_normal((2, 480, 12)) * 0.3 + 1.0
    z = O.trend_apply("detrend", y, rec, 2, 12)
    back = O.trend_apply("retrend", z, rec, 2, 12)
    assert np.abs(back - y).max() < 1e-12
