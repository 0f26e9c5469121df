"""CPU: the C-ABI library loads, exports every symbol include/sphemu_gpu.h
declares, and its host-only entry points (config validation, precision map)
behave like the reference — no GPU calls."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sphemu_gpu.h")).read()
    return sorted(set(re.findall(r"\b(sphemu_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol(sph):
    lib = sph._sphemu.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 20


def test_version(sph):
    assert sph.__version__ == "0.1.0"
    assert sph._sphemu.lib().sphemu_gpu_version().decode() == "0.1.0"


def test_precision_map_matches_oracle(sph, O):
    for v in ("dp", "dpsp", "dpsphp", "dphp"):
        for nt in (1, 4, 10, 33):
            for band in (1, 2):
                got = sph.assign_precisions(nt, v, band_width_dp=band, sp_fraction=0.07)
                want = O.assign_precisions(nt, variant=v, band_width_dp=band, sp_fraction=0.07)
                assert np.array_equal(got, want), (v, nt, band)


def test_config_validation_like_reference(sph):  # test_mpchol.cpp:263-280
    lib = sph._sphemu.lib()
    bad = [dict(tile_size=0), dict(workers=0), dict(sp_fraction=1.5), dict(band_width_dp=0)]
    for kw in bad:
        cfg = sph._sphemu.make_config(**kw)
        assert lib.sphemu_gpu_chol_config_validate(C.byref(cfg)) == 1
    assert lib.sphemu_gpu_chol_config_validate(C.byref(sph._sphemu.make_config())) == 0
    with pytest.raises(ValueError):
        sph._sphemu.make_config(variant="fp8")


def test_python_names_mirror_reference(sph):  # proj/python/sphemu/__init__.py
    for name in ("forward_sht", "inverse_sht", "tiled_cholesky", "make_spd_matrix", "max_band_limit",
                 "resolution_summary", "wigner_d_half_pi", "__version__"):
        assert hasattr(sph, name)
    assert sph.max_band_limit(721, 1440) == 720
    assert sph.max_band_limit(720, 1440) == 719
    s = sph.resolution_summary(720)
    assert s["grid_points"] == 719 * 1440 and abs(s["km_per_cell"] - 27.8) < 0.03
