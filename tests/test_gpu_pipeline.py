"""The train -> emulate pipeline (pipeline.cpp:18-54, stochastic.cpp:217-277)
through the Python Emulator drop-in (bindings/module.cpp:140-179, 232-243) on
the device, against the oracle's restatement of the same pipeline (C1's
chain: fit_trend -> detrend -> forward SHT -> fit_var -> covariance + nugget
-> factor -> noise field; emulate from the factor with the reference RNG).

Tolerances: trend records, u_hat, v2 1e-12 relative; lag coefficients 1e-10;
nugget the same escalation step (equal to the last bit or two); factor 1e-10; emulated fields 1e-9 relative (the same draws;
only summation order differs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.fixture(scope="module")
def small(O):
    x = O.synth_training_series(24, 48, 12, 60, 2, 91)
    return x, O.train(x, 2, 12, 2, 12, "dp", 64)


def test_train_matches_oracle(sph, O, small):
    x, m = small
    em = sph.Emulator.train(x, harmonics=2, period=12, var_order=2, band_limit=12, tile_size=64)
    assert em.band_limit == 12 and em.grid == (24, 48)
    assert rel(em.records, m["records"]) < 1e-12
    assert rel(em.phi, m["phi"]) < 1e-10
    assert rel(em.u_hat, m["u_hat"]) < 1e-12
    assert em.nugget == m["nugget"] and em.nugget > 0  # n = 116 < d = 144: nugget-regularised
    assert rel(em.factor(), m["v"]) < 1e-10
    assert rel(em.v2, m["v2"]) < 1e-12
    got = em.emulate(10, seed=42, replicates=3)
    want = O.emulate_model(m, 10, 42, 3)
    assert got.shape == want.shape == (3, 10, 24, 48)
    assert rel(got, want) < 1e-9
    # t_start shifts the trend phase only
    got5 = em.emulate(4, seed=7, replicates=1, t_start=5)
    want5 = O.emulate_model(m, 4, 7, 1, t_start=5)
    assert rel(got5, want5) < 1e-9


def test_default_band_limit_and_validation(sph, small):
    x, _ = small
    with pytest.raises(ValueError, match="resolve"):
        sph.Emulator.train(x, band_limit=40)
    with pytest.raises(ValueError, match="non-finite"):
        bad = x.copy()
        bad[0, 0, 0, 0] = np.nan
        sph.Emulator.train(bad, band_limit=12)
    with pytest.raises(ValueError, match="period"):
        sph.Emulator.train(x, period=7, band_limit=12)


def test_save_load_roundtrip(sph, small, tmp_path):
    x, _ = small
    em = sph.Emulator.train(x, harmonics=2, period=12, var_order=2, band_limit=12, tile_size=64)
    em.save(str(tmp_path))
    for name, magic in (("trend.bin", b"TRND"), ("var.bin", b"VARM"), ("ucov.bin", b"UCOV"), ("noise.bin", b"NOIS")):
        assert (tmp_path / name).read_bytes()[:4] == magic
    d = 144
    assert (tmp_path / "ucov.bin").stat().st_size == 4 + 4 + 8 + 8 * d * (d + 1) // 2 + 4 + 8 * d * (d + 1) // 2
    back = sph.Emulator.load(str(tmp_path))
    assert back.band_limit == 12 and back.grid == (24, 48) and back.nugget == em.nugget
    assert np.array_equal(back.records, em.records) and np.array_equal(back.phi, em.phi)
    assert np.array_equal(back.factor(), em.factor())
    assert np.array_equal(back.emulate(6, seed=3, replicates=2), em.emulate(6, seed=3, replicates=2))


def test_mixed_precision_factor_pipeline(sph, O, small):
    """A mixed-precision innovation factor (dpsphp) through the same pipeline:
    the tiles are quantized, emulation runs the tensor-core TRMM."""
    x, m = small
    em = sph.Emulator.train(x, harmonics=2, period=12, var_order=2, band_limit=12, tile_size=64, variant="dpsphp",
                            sp_fraction=0.3)
    v = em.factor()
    target = em.u_hat + em.nugget * np.eye(144)
    assert O.relative_residual(target, v) < 1e-2
    out = em.emulate(12, seed=5, replicates=2)
    assert np.isfinite(out).all()


@pytest.mark.slow
def test_c1_end_to_end(sph, O):
    """BASELINE configs[0] (C1): 180 x 360, L = 45, T = 100 daily steps,
    K = 2, period 365, P = 3, chol dp b = 256, then 10 replicates x 100 steps."""
    x = O.synth_training_series(180, 360, 45, 100, 1, 91, period=365)
    m = O.train(x, 2, 365, 3, 45, "dp", 256)
    em = sph.Emulator.train(x, harmonics=2, period=365, var_order=3, band_limit=45, tile_size=256)
    # same escalation step; 1e-8 mean(diag u_hat) differs in the last bit with the summation order
    assert abs(em.nugget - m["nugget"]) <= 1e-14 * m["nugget"]
    assert rel(em.records, m["records"]) < 1e-12
    assert rel(em.factor(), m["v"]) < 1e-10
    got = em.emulate(100, seed=42, replicates=10)
    want = O.emulate_model(m, 100, 42, 10)
    assert rel(got, want) < 1e-9
