"""SPHF field-series files (grid.cpp:69-106) — host only."""
import numpy as np
import pytest


def test_sphf_roundtrip(sph, tmp_path):
    a = np.random.default_rng(1).standard_normal((3, 5, 9, 16))
    p = str(tmp_path / "x.sphf")
    sph.write_sphf(p, a, 8)
    b, L = sph.read_sphf(p)
    assert L == 8 and np.array_equal(a, b)
    raw = open(p, "rb").read()
    assert raw[:4] == b"SPHF" and len(raw) == 4 + 6 * 4 + 8 * a.size
    sph.write_sphf(p, a[0])
    b, L = sph.read_sphf(p)
    assert L == 0 and b.shape == (5, 9, 16) and np.array_equal(a[0], b)


def test_sphf_rejects(sph, tmp_path):
    p = str(tmp_path / "y.sphf")
    with pytest.raises(ValueError, match="non-finite"):
        sph.write_sphf(p, np.full((2, 3, 4), np.nan))
    sph.write_sphf(p, np.zeros((2, 9, 16)), 8)
    open(p, "ab").write(b"x")
    with pytest.raises(RuntimeError, match="trailing"):
        sph.read_sphf(p)
    sph.write_sphf(p, np.zeros((2, 9, 16)), 12)  # L = 12 > max_band_limit(9, 16) = 8
    with pytest.raises(RuntimeError, match="band limit"):
        sph.read_sphf(p)
