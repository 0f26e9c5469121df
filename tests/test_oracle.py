"""CPU: the oracle against the reference's known-answer tests and against the
reference's own compiled code (oracle/_ref) / the committed golden vectors.
Test names cite the reference test they restate."""
import ctypes as C
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.npz")


@pytest.fixture(scope="module")
def G():
    return np.load(GOLDEN)


# ---- rng.hpp / half.hpp (bitwise) -----------------------------------------
def test_rng_stream_matches_reference(O, G):
    assert np.array_equal(O.normals(7, 2000), G["rng_normals_seed7"])


def test_half_quantization_matches_reference(O, G):
    sat = C.c_longlong(0)
    q = np.array([O.lib().so_quantize_half(float(x), C.byref(sat)) for x in G["half_in"]])
    assert np.array_equal(q, G["half_out"])
    assert sat.value == int(G["half_saturations"][0])


def test_quantize_kats(O):  # test_mpchol.cpp:177-202
    tile = np.array([1.0 / 3.0, 65505.0, -70000.0, 0.5])
    sp, c = O.quantize(tile, 1)
    assert sp[0] == float(np.float32(1.0 / 3.0)) and sp[3] == 0.5 and c.demotions_sp == 4
    hp, c = O.quantize(tile, 2)
    assert hp.tolist() == [0.333251953125, 65504.0, -65504.0, 0.5]
    assert c.demotions_hp == 4 and c.half_saturations == 1
    dp, c = O.quantize(tile, 0)
    assert np.array_equal(dp, tile)


# ---- mpchol (test_mpchol.cpp) ---------------------------------------------
def test_two_by_two_exact(O):  # :36-45
    for b in (1, 2):
        f, _ = O.tiled_cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]), tile_size=b)
        assert f.tolist() == [[2.0, 0.0], [1.0, math.sqrt(2.0)]]


def test_task_graph_counts(O):  # :47-71
    g = O.task_graph(4)
    assert len(g["kind"]) == 20 and np.bincount(g["kind"]).tolist() == [4, 6, 6, 4]
    assert len(g["succ"]) == int(g["indegree"].sum())
    assert int((g["indegree"] == 0).sum()) == 1 and g["kind"][0] == 0
    assert len(O.task_graph(1)["kind"]) == 1
    assert len(O.task_graph(8)["kind"]) == 8 + 28 + 28 + 56


def test_precision_map(O):  # :73-108
    nt = 10
    at = lambda m, i, j: m[i * (i + 1) // 2 + j]
    assert np.bincount(O.assign_precisions(nt, variant="dp"), minlength=3).tolist() == [55, 0, 0]
    assert np.bincount(O.assign_precisions(nt, variant="dpsp"), minlength=3).tolist() == [10, 45, 0]
    assert np.bincount(O.assign_precisions(nt, variant="dphp"), minlength=3).tolist() == [10, 0, 45]
    m = O.assign_precisions(nt, variant="dpsphp", sp_fraction=0.05)
    assert np.bincount(m, minlength=3).tolist() == [10, 3, 42]
    assert [at(m, 1, 0), at(m, 2, 1), at(m, 3, 2), at(m, 4, 3), at(m, 2, 0)] == [1, 1, 1, 2, 2]
    w = O.assign_precisions(nt, variant="dpsp", band_width_dp=2)
    assert np.bincount(w, minlength=3).tolist() == [19, 36, 0]


@pytest.mark.parametrize("n", [96, 100])
def test_dp_factor_matches_untiled(O, n):  # :110-121
    a = O.make_spd(n, 3)
    f, _ = O.tiled_cholesky(a, tile_size=32)
    assert np.abs(f - O.dense_cholesky(a)).max() < 1e-13
    assert O.relative_residual(a, f) < 1e-14


def test_benchmark_matrix_shape(O):  # :123-140
    a = O.make_spd(64, 11)
    assert np.array_equal(a, a.T)
    d = np.diag(a)
    assert (d > 0).all() and ((np.abs(a).sum(1) - d) < 10 * d).all()
    assert np.array_equal(O.make_spd(64, 11), a) and not np.array_equal(O.make_spd(64, 12), a)


def test_indefinite_names_failing_tile(O):  # :142-154
    a = np.eye(96)
    a[40, 40] = -1.0
    with pytest.raises(O.NotPositiveDefinite) as e:
        O.tiled_cholesky(a, tile_size=32)
    assert e.value.tile_index == 1


def test_worker_invariance(O):  # :156-175
    a = O.make_spd(256, 7)
    s, ss = O.tiled_cholesky(a, "dpsphp", 32, workers=1, sp_fraction=0.2)
    t, ts = O.tiled_cholesky(a, "dpsphp", 32, workers=4, sp_fraction=0.2)
    assert np.array_equal(s, t) and ss["conversions"] == ts["conversions"] and ts["workers"] == 4


def test_residual_thresholds_monotone(O):  # :219-234
    a = O.make_spd(256, 5)
    r = [O.relative_residual(a, O.tiled_cholesky(a, v, 32)[0]) for v in ("dp", "dpsp", "dpsphp", "dphp")]
    assert r[0] < 1e-13 and r[1] < 5e-6 and r[2] < 1e-2 and r[3] < 5e-2
    assert r[0] <= r[1] <= r[2] <= r[3]


def test_stats_footprint(O):  # :236-261
    _, s = O.tiled_cholesky(O.make_spd(256, 9), "dpsp", 64)
    assert s["n_tiles"] == 4 and s["tasks"] == {"potrf": 4, "trsm": 6, "syrk": 6, "gemm": 4, "total": 20}
    assert s["tiles"]["dp"] == 4 and s["tiles"]["sp"] == 6
    assert s["bytes"]["dp"] == 4 * 64 * 64 * 8 and s["bytes"]["sp"] == 6 * 64 * 64 * 4
    assert s["conversions"]["to_sp"] > 0


# ---- wigner (test_wigner.cpp, wigner.cpp) ----------------------------------
def test_wigner_closed_forms(O):  # test_wigner.cpp:23-31
    b = O.lib().so_wigner_brute
    assert b(0, 0, 0) == pytest.approx(1.0, rel=1e-15)
    assert b(1, 1, 1) == pytest.approx(0.5, rel=1e-14)
    assert b(1, 1, -1) == pytest.approx(0.5, rel=1e-14)
    assert abs(b(1, 0, 0)) < 1e-15
    assert b(1, 1, 0) == pytest.approx(-1 / math.sqrt(2), rel=1e-14)
    assert b(2, 2, 0) == pytest.approx(math.sqrt(3 / 8), rel=1e-14)
    assert b(2, 0, 0) == pytest.approx(-0.5, rel=1e-14)


def test_wigner_recursion_vs_factorial_sum(O):  # test_wigner.cpp:33-43
    w = O.Wigner(13)
    worst = max(abs(w.d(l, m2, m) - O.lib().so_wigner_brute(l, m2, m))
                for l in range(13) for m2 in range(-l, l + 1) for m in range(-l, l + 1))
    assert worst < 1e-12


@pytest.mark.parametrize("L", [13, 33])
def test_wigner_tables_match_reference(O, G, L):
    w = O.Wigner(L)
    d = np.array([w.d(l, m2, m) for l in range(L) for m2 in range(-l, l + 1) for m in range(-l, l + 1)])
    q = np.array([w.q(l, m, m2) for l in range(L) for m in range(l + 1) for m2 in range(L)])
    assert np.array_equal(d, G[f"wigner_d_L{L}"]) and np.array_equal(q, G[f"wigner_q_L{L}"])


def test_wigner_q_and_cap(O):  # test_wigner.cpp:61-73, 306-308
    w = O.Wigner(4)
    assert w.q(0, 0, 0) == pytest.approx(0.2820947917738781, rel=1e-14)
    assert w.q(1, 0, 1) == pytest.approx(math.sqrt(3 / (4 * math.pi)) * 0.5, rel=1e-14)
    assert w.q(1, 1, 3) == 0.0
    with pytest.raises(ValueError):
        O.Wigner(512, cap=1024)
    assert O.lib().so_wigner_bytes(720) > (2 << 30)


# ---- sht (test_sht.cpp) ------------------------------------------------------
def test_line_integrals(O):  # test_sht.cpp:51-59
    def I(q):
        re, im = C.c_double(), C.c_double()
        O.lib().so_i_integral(q, C.byref(re), C.byref(im))
        return complex(re.value, im.value)
    assert I(0) == 2 and I(1) == complex(0, math.pi / 2) and I(-1) == complex(0, -math.pi / 2)
    assert I(2) == -2 / 3 and I(3) == 0 and I(4) == -2 / 15 and I(-2) == -2 / 3


@pytest.mark.parametrize("grid", [(9, 16, 8), (33, 64, 16), (17, 20, 9), (46, 90, 45)])
def test_sht_matches_reference(O, G, grid):
    nt, nphi, L = grid
    key = f"sht_{nt}x{nphi}_L{L}"
    P = O.Plan(nt, nphi, L)
    assert np.array_equal(P.inverse(G[key + "_coeffs"]), G[key + "_fields"])
    assert np.array_equal(P.forward(G[key + "_x"]), G[key + "_fx"])


def test_constant_field(O):  # test_sht.cpp:72-83
    P = O.Plan(7, 12, 6)
    c = P.forward(np.full((7, 12), 2.5))[0]
    assert c[0] == pytest.approx(2.5 * math.sqrt(4 * math.pi), rel=1e-13)
    assert np.abs(c[1:]).max() < 1e-12
    assert np.allclose(P.inverse(c)[0], 2.5, rtol=1e-13)


def test_round_trip_and_parseval(O):  # test_sht.cpp:85-102,135-143; acceptance_main.cpp:86-109
    for L in (8, 16, 32):
        P = O.Plan(L + 1, 2 * L, L)
        for rep in range(1, 4):
            c = O.draw_random_coefficients(L, 100 * L + rep)
            f = P.inverse(c)
            assert np.abs(P.forward(f)[0] - c).max() < 1e-10
            e_c = O.lib().so_parseval_energy(c, L)
            e_f = O.lib().so_field_energy_quadrature(np.ascontiguousarray(f[0]), L + 1, 2 * L)
            assert abs(e_c - e_f) / e_c < 1e-8


def test_direct_synthesis_matches(O):  # test_sht.cpp:145-152
    P = O.Plan(7, 12, 6)
    c = O.draw_random_coefficients(6, 13)
    d = np.empty((7, 12))
    O.lib().so_synth_bandlimited(c, 6, 7, 12, d)
    assert np.abs(P.inverse(c)[0] - d).max() < 1e-9


@pytest.mark.parametrize("grid", [(7, 12, 6), (9, 16, 16), (21, 40, 45), (121, 256, 20)])
def test_synth_bandlimited_matches_reference_golden(O, grid):  # sht.cpp:435-466 via oracle/_ref
    nt, nphi, L = grid
    G = np.load(GOLDEN)
    key = f"synth_{nt}x{nphi}_L{L}"
    d = np.empty((nt, nphi))
    O.lib().so_synth_bandlimited(G[key + "_coeffs"], L, nt, nphi, d)
    assert np.array_equal(d, G[key + "_field"])


def test_batch_thread_invariance(O):  # test_sht.cpp:163-181
    P = O.Plan(11, 20, 10)
    f = P.inverse(np.stack([O.draw_random_coefficients(10, 100 + s) for s in range(14)]))
    assert np.array_equal(P.forward(f, threads=1), P.forward(f, threads=3))


def test_plan_rejects_unresolvable(O):  # test_sht.cpp:196-199
    with pytest.raises(ValueError):
        O.Plan(9, 16, 9)
    O.Plan(9, 16, 8)


# ---- oracle/_ref itself (when built from /root/reference here) ------------
@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "libsphemu_ref.so")),
                    reason="oracle/_ref not built")
def test_oracle_bitwise_vs_reference_sources(O):
    R = O.ref()
    for (nt, nphi, L) in ((13, 24, 12), (21, 40, 20)):
        c = np.stack([O.draw_random_coefficients(L, s) for s in range(3)])
        f2 = np.empty((3, nt, nphi))
        R.ref_inverse_sht_batch(nt, nphi, L, c, 3, f2, 2)
        P = O.Plan(nt, nphi, L)
        assert np.array_equal(P.inverse(c), f2)
        g2 = np.empty((3, L * L))
        R.ref_forward_sht_batch(nt, nphi, L, f2, 3, g2, 2)
        assert np.array_equal(P.forward(f2), g2)
