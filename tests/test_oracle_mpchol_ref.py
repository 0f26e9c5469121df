"""The oracle's restatement of mpchol.cpp (oracle/so_mpchol.c, the checker
of every Cholesky parity test) pinned to the reference's OWN mpchol.cpp,
compiled in place from /root/reference (oracle/ref/build_ref.sh) against a
minimal Eigen stand-in whose three kernels follow so_mpchol.c's loop order:
the reference's precision map, task graph and scheduler, input and
per-task quantization, POTRF, statistics JSON and NotPositiveDefiniteError
must reproduce the oracle bitwise. Host only; skipped where the reference
sources are absent (the GPU box)."""
import json

import numpy as np
import pytest


@pytest.fixture(scope="module")
def R(O):
    if O.ref_mpchol() is None:
        pytest.skip("reference mpchol.cpp not built here (no /root/reference)")
    O.lib().so_use_blas(None)  # the oracle's loop kernels (the shim's order)
    return O


@pytest.mark.parametrize("variant", ["dp", "dpsp", "dpsphp", "dphp"])
@pytest.mark.parametrize("n,b,workers", [(100, 32, 1), (256, 32, 4), (300, 64, 3)])
def test_factor_and_stats_bitwise(R, variant, n, b, workers):
    a = R.make_spd(n, 7)
    rc, f_ref, js, _ = R.ref_tiled_cholesky(a, variant, b, workers, 1, 0.2)
    assert rc == 0, js
    f, st = R.tiled_cholesky(a, variant, tile_size=b, workers=workers, sp_fraction=0.2)
    assert np.array_equal(f, f_ref)
    ref_stats = json.loads(js)
    mine = json.loads(R.stats_json(st))
    for key in ("n", "tile_size", "n_tiles", "workers", "variant", "tasks", "tiles", "bytes", "conversions"):
        assert mine[key] == ref_stats[key], key


def test_dense_input_and_band(R):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((400, 200))
    a = x.T @ x / 400 + 1e-3 * np.eye(200)
    for variant in ("dpsp", "dpsphp"):
        rc, f_ref, js, _ = R.ref_tiled_cholesky(a, variant, 48, 2, 2, 0.3)
        f, _ = R.tiled_cholesky(a, variant, tile_size=48, workers=2, band_width_dp=2, sp_fraction=0.3)
        assert rc == 0 and np.array_equal(f, f_ref)


def test_precision_map_and_generator(R):
    import ctypes as C
    for variant, band, sp in (("dpsphp", 1, 0.05), ("dpsphp", 2, 0.3), ("dphp", 1, 0.05), ("dpsp", 3, 0.05)):
        for nt in (1, 4, 10, 31):
            out = np.zeros(nt * (nt + 1) // 2, dtype=np.uint8)
            R.ref_mpchol().ref_assign_precisions(nt, R.VARIANTS[variant], band, sp, out.ctypes.data)
            assert np.array_equal(out, R.assign_precisions(nt, variant=variant, band_width_dp=band, sp_fraction=sp))
    a = np.empty((300, 300))
    R.ref_mpchol().ref_make_spd(300, C.c_uint64(5), a.ctypes.data)
    assert np.array_equal(a, R.make_spd(300, 5))


def test_not_positive_definite_tile_and_message(R):
    a = np.eye(96)
    a[40, 40] = -1.0
    rc, _, msg, tile = R.ref_tiled_cholesky(a, "dp", 32)
    assert rc == 1 and tile == 1 and "non-positive pivot" in msg
    with pytest.raises(R.NotPositiveDefinite) as e:
        R.tiled_cholesky(a, "dp", tile_size=32)
    assert e.value.tile_index == tile
