"""GPU mean structure (trend.cu: mean_table / detrend / retrend, trend.cpp:252-324)
against the oracle restatement: bitwise (explicit round-to-nearest, no FMA
contraction, the same libm cos/sin for the per-step scalars), including the
forcing terms, ragged location blocks, many row blocks and the error paths."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def records(points, k, seed=1, lag=0.0):
    rng = np.random.default_rng(seed)
    rec = rng.standard_normal((points, 5 + 2 * k))
    rec[:, 2] = lag
    rec[:, 3] = 0.6
    rec[:, -1] = 0.5 + rng.random(points)
    return rec


@pytest.mark.parametrize("points,k,period,t_len,t_start", [
    (12, 1, 12, 24, 13),        # test_trend.cpp:195-206
    (181 * 360, 5, 8760, 70, 8700),  # ragged last CTA, year boundary
    (1, 0, 365, 1, 1),
    (300, 2, 12, 1000, 5),      # many row blocks
])
def test_mean_table_bitwise(sph, O, points, k, period, t_len, t_start):
    rec = records(points, k)
    got = sph.mean_table(rec, k, period, t_len, t_start)
    want = O.mean_table(rec, k, period, t_len, t_start)
    assert np.array_equal(got, want)


def test_mean_table_with_forcing_bitwise(sph, O):
    rec = records(777, 2, lag=0.3)
    x = np.linspace(0.1, 2.0, 6)
    hist = np.array([0.05, 0.02, 0.01])
    got = sph.mean_table(rec, 2, 12, 60, 1, forcing=sph.ForcingTrajectory(x, hist))
    want = O.mean_table(rec, 2, 12, 60, 1, forcing=(x, hist))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("r_len,t_len,points", [(1, 24, 12), (3, 48, 91 * 180), (2, 5, 129)])
def test_detrend_retrend_bitwise(sph, O, r_len, t_len, points):
    rec = records(points, 2, seed=7)
    y = np.random.default_rng(9).standard_normal((r_len, t_len, points)) + 2.0
    z = sph.detrend(y, rec, 2, 12, t_start=3)
    assert np.array_equal(z, O.trend_apply("detrend", y, rec, 2, 12, None, 3))
    back = sph.retrend(z, rec, 2, 12, t_start=3)
    assert np.array_equal(back, O.trend_apply("retrend", z, rec, 2, 12, None, 3))
    assert np.abs(back - y).max() < 1e-12  # test_trend.cpp:165-178


def test_errors(sph):
    with pytest.raises(ValueError, match="1-based"):
        sph.mean_table(records(4, 1), 1, 12, 3, 0)
    with pytest.raises(ValueError, match="history"):
        sph.mean_table(records(4, 0, lag=0.5), 0, 12, 12, 1, forcing=(np.array([1.0]), None))
    with pytest.raises(ValueError):
        sph.detrend(np.zeros((1, 4, 5)), records(4, 1), 1, 12)
    assert sph.mean_table(records(4, 1), 1, 12, 0, 1).shape == (0, 4)


def test_device_records_match_host(sph, O):
    """records may be a device pointer (detected): only the lag column and rho
    cross PCIe; results identical to the host-records call."""
    import ctypes as C

    import torch
    rec = records(5000, 3, lag=0.2)
    x, hist = np.linspace(0.1, 1.0, 4), np.array([0.05])
    y = np.random.default_rng(2).standard_normal((2, 30, 5000))
    want = sph.retrend(y, rec, 3, 12, forcing=(x, hist), t_start=2)
    d_rec = torch.from_numpy(rec).cuda()
    lib = sph._sphemu.lib()
    out = np.empty_like(y)
    vp = C.c_void_p
    rc = lib.sphemu_gpu_retrend(vp(y.ctypes.data), 0, 2, 30, vp(d_rec.data_ptr()), 5000, 3, 12, vp(x.ctypes.data),
                                4, vp(hist.ctypes.data), 1, 2, vp(out.ctypes.data), 0)
    assert rc == 0, lib.sphemu_gpu_last_error()
    assert np.array_equal(out, want)
    assert np.array_equal(want, O.trend_apply("retrend", y, rec, 3, 12, (x, hist), 2))
