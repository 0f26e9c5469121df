"""ctypes bindings for the CPU oracle (liboracle.so) and oracle/_ref.

TEST INFRASTRUCTURE: imported only by tests/, __graft_entry__.smoke() and
bench.py's cpu-baseline / --impl reference leg. Never part of the product path.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsphemu_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")

VARIANTS = {"dp": 0, "dpsp": 1, "dpsphp": 2, "dphp": 3}


class CholConfig(C.Structure):
    _fields_ = [("variant", C.c_int), ("tile_size", C.c_int), ("band_width_dp", C.c_int),
                ("sp_fraction", C.c_double), ("workers", C.c_int), ("hp_format", C.c_int)]


class Counters(C.Structure):
    _fields_ = [("demotions_sp", C.c_int64), ("demotions_hp", C.c_int64),
                ("half_saturations", C.c_int64)]


class CholStats(C.Structure):
    _fields_ = [("n", C.c_int), ("tile_size", C.c_int), ("n_tiles", C.c_int), ("workers", C.c_int),
                ("variant", C.c_int), ("tasks_potrf", C.c_int64), ("tasks_trsm", C.c_int64),
                ("tasks_syrk", C.c_int64), ("tasks_gemm", C.c_int64), ("tiles_dp", C.c_int64),
                ("tiles_sp", C.c_int64), ("tiles_hp", C.c_int64), ("bytes_dp", C.c_int64),
                ("bytes_sp", C.c_int64), ("bytes_hp", C.c_int64), ("conv", Counters),
                ("wall_seconds", C.c_double)]

    def as_dict(self) -> dict:
        names = ["dp", "dpsp", "dpsphp", "dphp"]
        return {
            "n": self.n, "tile_size": self.tile_size, "n_tiles": self.n_tiles,
            "workers": self.workers, "variant": names[self.variant],
            "tasks": {"potrf": self.tasks_potrf, "trsm": self.tasks_trsm, "syrk": self.tasks_syrk,
                      "gemm": self.tasks_gemm,
                      "total": self.tasks_potrf + self.tasks_trsm + self.tasks_syrk + self.tasks_gemm},
            "tiles": {"dp": self.tiles_dp, "sp": self.tiles_sp, "hp": self.tiles_hp},
            "bytes": {"dp": self.bytes_dp, "sp": self.bytes_sp, "hp": self.bytes_hp,
                      "total": self.bytes_dp + self.bytes_sp + self.bytes_hp},
            "conversions": {"to_sp": self.conv.demotions_sp, "to_hp": self.conv.demotions_hp,
                            "half_saturations": self.conv.half_saturations},
            "wall_seconds": self.wall_seconds,
        }


class NotPositiveDefinite(RuntimeError):
    def __init__(self, tile_index: int):
        super().__init__(f"diagonal tile {tile_index} has a non-positive pivot")
        self.tile_index = tile_index


def build(force: bool = False) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    if force or not os.path.exists(LIB_PATH) or _stale():
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    if os.path.isdir(os.environ.get("SPHEMU_REFERENCE", "/root/reference/proj")) and (
            force or not os.path.exists(REF_PATH) or not os.path.exists(os.path.join(HERE, "_ref",
                                                                                      "libsphemu_ref_mpchol.so"))):
        subprocess.run([os.path.join(HERE, "ref", "build_ref.sh")], check=True)


def _stale() -> bool:
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in os.listdir(HERE)
               if f.endswith((".c", ".h")))


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.so_rng_normals.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.so_quantize_half.argtypes = [C.c_double, C.POINTER(C.c_longlong)]
        L.so_quantize_half.restype = C.c_double
        L.so_quantize_bf16.argtypes = [C.c_double, C.POINTER(C.c_longlong)]
        L.so_quantize_bf16.restype = C.c_double
        L.so_quantize_tile.argtypes = [_dp, C.c_int64, C.c_int, C.c_int, C.POINTER(Counters)]
        L.so_assign_precisions.argtypes = [C.c_int, C.POINTER(CholConfig), _u8]
        L.so_task_count.argtypes = [C.c_int]
        L.so_task_count.restype = C.c_int64
        L.so_task_graph.restype = C.c_int64
        L.so_tiled_cholesky_dense.argtypes = [_dp, C.c_int, C.POINTER(CholConfig), _dp,
                                              C.POINTER(CholStats), C.POINTER(C.c_int)]
        L.so_make_spd.argtypes = [C.c_int, C.c_uint64, _dp]
        L.so_make_spd_factors.argtypes = [C.c_int, C.c_uint64, _dp, _dp]
        L.so_dense_cholesky.argtypes = [_dp, C.c_int, _dp]
        L.so_relative_residual.argtypes = [_dp, _dp, C.c_int, C.c_int]
        L.so_relative_residual.restype = C.c_double
        L.so_use_blas.argtypes = [C.c_char_p]
        L.so_i_integral.argtypes = [C.c_longlong, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.so_wigner_build.argtypes = [C.c_int, C.c_size_t]
        L.so_wigner_build.restype = C.c_void_p
        L.so_wigner_free.argtypes = [C.c_void_p]
        L.so_wigner_d.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.so_wigner_d.restype = C.c_double
        L.so_wigner_q.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.so_wigner_q.restype = C.c_double
        L.so_wigner_renorm_warnings.argtypes = [C.c_void_p]
        L.so_wigner_bytes.argtypes = [C.c_int]
        L.so_wigner_bytes.restype = C.c_size_t
        L.so_wigner_brute.argtypes = [C.c_int, C.c_int, C.c_int]
        L.so_wigner_brute.restype = C.c_double
        L.so_plan_build.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.so_plan_build.restype = C.c_void_p
        L.so_plan_free.argtypes = [C.c_void_p]
        L.so_forward_sht_batch.argtypes = [C.c_void_p, _dp, C.c_int64, _dp, C.c_int]
        L.so_inverse_sht_batch.argtypes = [C.c_void_p, _dp, C.c_int64, _dp, C.c_int]
        L.so_normalized_legendre_all.argtypes = [C.c_int, C.c_double, _dp]
        L.so_synth_bandlimited.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp]
        L.so_draw_random_coefficients.argtypes = [C.c_int, C.c_uint64, _dp]
        L.so_field_energy_quadrature.argtypes = [_dp, C.c_int, C.c_int]
        L.so_field_energy_quadrature.restype = C.c_double
        L.so_parseval_energy.argtypes = [_dp, C.c_int]
        L.so_parseval_energy.restype = C.c_double
        L.so_dft.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.so_estimate_innovation_covariance.argtypes = [
            _dp, C.c_int64, C.c_int, C.POINTER(CholConfig), C.c_int, _dp, _dp,
            C.POINTER(C.c_double), C.POINTER(CholStats)]
        L.so_emulate.argtypes = [C.c_void_p, _dp, C.c_int, _dp, C.c_int, _dp, _dp, _dp, C.c_int,
                                 C.c_uint64, C.c_int, C.c_int, _dp]
        L.so_eval_mean_trend.restype = C.c_double
        L.so_eval_mean_trend.argtypes = [_dp, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                         C.c_void_p, C.c_int64, C.POINTER(C.c_int)]
        L.so_mean_table.argtypes = [_dp, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                    C.c_int64, C.c_int, C.c_int64, _dp]
        L.so_trend_apply.argtypes = [C.c_int, _dp, C.c_int, C.c_int, _dp, C.c_int64, C.c_int, C.c_int,
                                     C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, _dp]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


REF_MPCHOL_PATH = os.path.join(HERE, "_ref", "libsphemu_ref_mpchol.so")
_ref_mpchol = None


def ref_mpchol():
    """The reference's own mpchol.cpp over the Eigen shim (oracle/_ref), or None."""
    global _ref_mpchol
    if _ref_mpchol is None and os.path.exists(REF_MPCHOL_PATH):
        R = C.CDLL(REF_MPCHOL_PATH)
        R.ref_tiled_cholesky_dense.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                               C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
        R.ref_assign_precisions.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p]
        R.ref_make_spd.argtypes = [C.c_int, C.c_uint64, C.c_void_p]
        _ref_mpchol = R
    return _ref_mpchol


def ref_tiled_cholesky(a, variant="dp", tile_size=128, workers=1, band_width_dp=1, sp_fraction=0.05):
    """mpchol.cpp's tiled_cholesky_dense itself: (rc, factor, stats_json_or_message, failed_tile)."""
    R = ref_mpchol()
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    out = np.zeros_like(a)
    buf = C.create_string_buffer(1 << 14)
    failed = C.c_int(-1)
    rc = R.ref_tiled_cholesky_dense(a.ctypes.data, n, VARIANTS[variant], tile_size, workers, band_width_dp,
                                    sp_fraction, out.ctypes.data, buf, len(buf), C.byref(failed))
    return rc, out, buf.value.decode(), failed.value


def ref():
    """The reference's own wigner/grid/sht/half/rng code (oracle/_ref)."""
    global _ref
    if _ref is None:
        R = C.CDLL(REF_PATH)
        R.ref_quantize_half.argtypes = [C.c_double, C.POINTER(C.c_longlong)]
        R.ref_quantize_half.restype = C.c_double
        R.ref_rng_normals.argtypes = [C.c_uint64, C.c_int64, _dp]
        R.ref_rng_uniforms.argtypes = [C.c_uint64, C.c_int64, _dp]
        R.ref_i_integral.argtypes = [C.c_longlong, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        R.ref_wigner_dump.argtypes = [C.c_int, _dp, _dp, C.POINTER(C.c_int)]
        R.ref_wigner_check_cap.argtypes = [C.c_int, C.c_size_t]
        R.ref_wigner_brute.argtypes = [C.c_int, C.c_int, C.c_int]
        R.ref_wigner_brute.restype = C.c_double
        R.ref_forward_sht_batch.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int64, _dp, C.c_int]
        R.ref_inverse_sht_batch.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int64, _dp, C.c_int]
        R.ref_forward_sht_via_weights.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp]
        R.ref_draw_random_coefficients.argtypes = [C.c_int, C.c_uint64, _dp]
        R.ref_synth_bandlimited.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _dp]
        R.ref_normalized_legendre_all.argtypes = [C.c_int, C.c_double, _dp]
        R.ref_field_energy_quadrature.argtypes = [_dp, C.c_int, C.c_int]
        R.ref_field_energy_quadrature.restype = C.c_double
        _ref = R
    return _ref


# ----------------------------------------------------------------------------
# numpy-level helpers
# ----------------------------------------------------------------------------

def config(variant="dp", tile_size=128, band_width_dp=1, sp_fraction=0.05, workers=1,
           hp_format="fp16") -> CholConfig:
    return CholConfig(VARIANTS[variant] if isinstance(variant, str) else variant, tile_size,
                      band_width_dp, sp_fraction, workers, 1 if hp_format == "bf16" else 0)


def normals(seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    lib().so_rng_normals(seed, n, out)
    return out


def make_spd(n: int, seed: int = 1) -> np.ndarray:
    a = np.empty((n, n))
    lib().so_make_spd(n, seed, a)
    return a


def spd_factors(n: int, seed: int = 1):
    d = np.empty(n)
    pw = np.empty(n)
    lib().so_make_spd_factors(n, seed, d, pw)
    return d, pw


def assign_precisions(n_tiles: int, **kw) -> np.ndarray:
    out = np.empty(n_tiles * (n_tiles + 1) // 2, dtype=np.uint8)
    rc = lib().so_assign_precisions(n_tiles, C.byref(config(**kw)), out)
    if rc:
        raise ValueError("invalid configuration")
    return out


def task_graph(n_tiles: int):
    cnt = lib().so_task_count(n_tiles)
    kind = np.empty(cnt, dtype=np.uint8)
    ti, tj, tk, indeg = (np.empty(cnt, dtype=np.int32) for _ in range(4))
    off = np.empty(cnt + 1, dtype=np.int64)
    cap = 8 * cnt + 16
    succ = np.empty(cap, dtype=np.int32)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    lib().so_task_graph.argtypes = [C.c_int] + [C.c_void_p] * 7 + [C.c_int64]
    edges = lib().so_task_graph(n_tiles, ptr(kind), ptr(ti), ptr(tj), ptr(tk), ptr(off),
                                ptr(succ), ptr(indeg), cap)
    return dict(kind=kind, i=ti, j=tj, k=tk, succ_off=off, succ=succ[:edges], indegree=indeg)


def quantize(x: np.ndarray, prec: int, hp_format="fp16"):
    y = np.ascontiguousarray(x, dtype=np.float64).copy()
    c = Counters()
    lib().so_quantize_tile(y, y.size, prec, 1 if hp_format == "bf16" else 0, C.byref(c))
    return y, c


def tiled_cholesky(a: np.ndarray, variant="dp", tile_size=128, workers=1, band_width_dp=1,
                   sp_fraction=0.05, hp_format="fp16", precision_map=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    out = np.empty_like(a)
    st = CholStats()
    failed = C.c_int(-1)
    cfg = config(variant, tile_size, band_width_dp, sp_fraction, workers, hp_format)
    if precision_map is not None:
        pm = np.ascontiguousarray(precision_map, dtype=np.uint8)
        lib().so_tiled_cholesky_dense_map.argtypes = [C.c_void_p, C.c_int, C.POINTER(CholConfig), C.c_void_p,
                                                      C.c_void_p, C.POINTER(CholStats), C.POINTER(C.c_int)]
        rc = lib().so_tiled_cholesky_dense_map(a.ctypes.data, n, C.byref(cfg), pm.ctypes.data, out.ctypes.data,
                                               C.byref(st), C.byref(failed))
    else:
        rc = lib().so_tiled_cholesky_dense(a, n, C.byref(cfg), out, C.byref(st), C.byref(failed))
    if rc == 1:
        raise NotPositiveDefinite(failed.value)
    if rc:
        raise ValueError("invalid configuration")
    return out, st.as_dict()


def dense_cholesky(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty_like(a)
    if lib().so_dense_cholesky(a, a.shape[0], out):
        raise RuntimeError("matrix is not positive definite")
    return out


def relative_residual(a: np.ndarray, l: np.ndarray, threads: int = 0) -> float:
    threads = threads or os.cpu_count() or 1
    return lib().so_relative_residual(np.ascontiguousarray(a), np.ascontiguousarray(l),
                                      a.shape[0], threads)


class Wigner:
    def __init__(self, band_limit: int, cap: int = 2 << 30):
        self.L = band_limit
        self.h = lib().so_wigner_build(band_limit, cap)
        if not self.h:
            raise ValueError("Wigner tables over the memory cap")

    def __del__(self):
        if getattr(self, "h", None):
            lib().so_wigner_free(self.h)

    def d(self, l, m2, m):
        return lib().so_wigner_d(self.h, l, m2, m)

    def q(self, l, m, m2):
        return lib().so_wigner_q(self.h, l, m, m2)

    @property
    def renorm_warnings(self):
        return lib().so_wigner_renorm_warnings(self.h)


class Plan:
    def __init__(self, n_theta: int, n_phi: int, band_limit: int):
        self.n_theta, self.n_phi, self.L = n_theta, n_phi, band_limit
        self.h = lib().so_plan_build(n_theta, n_phi, band_limit, None)
        if not self.h:
            raise ValueError(f"grid {n_theta}x{n_phi} does not resolve band limit {band_limit}")

    def __del__(self):
        if getattr(self, "h", None):
            lib().so_plan_free(self.h)

    def forward(self, fields: np.ndarray, threads: int = 1) -> np.ndarray:
        f = np.ascontiguousarray(fields, dtype=np.float64).reshape(-1, self.n_theta * self.n_phi)
        out = np.empty((f.shape[0], self.L * self.L))
        lib().so_forward_sht_batch(self.h, f, f.shape[0], out, threads)
        return out

    def inverse(self, coeffs: np.ndarray, threads: int = 1) -> np.ndarray:
        c = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1, self.L * self.L)
        out = np.empty((c.shape[0], self.n_theta, self.n_phi))
        lib().so_inverse_sht_batch(self.h, c, c.shape[0], out, threads)
        return out


def draw_random_coefficients(band_limit: int, seed: int) -> np.ndarray:
    out = np.empty(band_limit * band_limit)
    lib().so_draw_random_coefficients(band_limit, seed, out)
    return out


def emulate(plan: Plan, v, phi, means, sigma, v2, t_out, seed, r_len=1, threads=1):
    d = v.shape[0]
    order = 0 if phi is None else phi.shape[0]
    phi_a = np.ascontiguousarray(phi if order else np.zeros((1, d)), dtype=np.float64)
    out = np.empty((r_len, t_out, plan.n_theta, plan.n_phi))
    lib().so_emulate(plan.h, np.ascontiguousarray(v), d, phi_a, order,
                     np.ascontiguousarray(means), np.ascontiguousarray(sigma),
                     np.ascontiguousarray(v2), t_out, seed, r_len, threads, out)
    return out


def stats_json(stats: dict) -> str:
    return json.dumps(stats, indent=2) + "\n"


def find_openblas():
    """scipy's bundled OpenBLAS: the oracle's stand-in for Eigen's tile BLAS."""
    try:
        import scipy  # noqa: F401
        d = os.path.join(os.path.dirname(os.path.dirname(scipy.__file__)), "scipy.libs")
        for f in sorted(os.listdir(d)):
            if f.startswith("libscipy_openblas") and f.endswith(".so"):
                return os.path.join(d, f)
    except Exception:
        pass
    return None


def _forcing(forcing):
    x, h = forcing if forcing is not None else (None, None)
    x = np.ascontiguousarray(np.zeros(0) if x is None else x, dtype=np.float64)
    h = np.ascontiguousarray(np.zeros(0) if h is None else h, dtype=np.float64)
    return (x, h), [x.ctypes.data if x.size else None, x.size, h.ctypes.data if h.size else None, h.size]


def eval_mean_trend(records, harmonics, period, loc, t, forcing=None):
    """eval_mean_trend (trend.cpp:65-83); raises ValueError on missing lag history."""
    keep, fa = _forcing(forcing)
    err = C.c_int()
    v = lib().so_eval_mean_trend(np.ascontiguousarray(records, dtype=np.float64), harmonics, period, loc, t,
                                 *fa, C.byref(err))
    if err.value:
        raise ValueError("lagged forcing term needs history")
    return v


def mean_table(records, harmonics, period, t_len, t_start=1, forcing=None):
    """mean_table (trend.cpp:252-287): (t_len, points)."""
    rec = np.ascontiguousarray(records, dtype=np.float64)
    points = rec.size // (5 + 2 * harmonics)
    keep, fa = _forcing(forcing)
    out = np.empty((t_len, points))
    rc = lib().so_mean_table(rec, points, harmonics, period, *fa, t_len, t_start, out)
    if rc:
        raise ValueError("time steps are 1-based" if rc == -1 else "lagged forcing term needs history")
    return out


def trend_apply(mode, series, records, harmonics, period, forcing=None, t_start=1):
    """mode "detrend" (trend.cpp:289-305) or "retrend" (trend.cpp:307-324) over (r, t, points)."""
    rec = np.ascontiguousarray(records, dtype=np.float64)
    points = rec.size // (5 + 2 * harmonics)
    x = np.ascontiguousarray(series, dtype=np.float64).reshape(-1, series.shape[-2] if series.ndim == 3 else
                                                               series.shape[0], points)
    keep, fa = _forcing(forcing)
    out = np.empty(x.shape)
    rc = lib().so_trend_apply({"detrend": 0, "retrend": 1}[mode], x, x.shape[0], x.shape[1], rec, points,
                              harmonics, period, *fa, t_start, out)
    if rc:
        raise ValueError("time steps are 1-based" if rc == -1 else "lagged forcing term needs history")
    return out.reshape(series.shape)


def _fullpiv_rank(a, threshold=1e-13):
    """Rank of Eigen's FullPivLU with setThreshold(threshold) (stochastic.cpp:72-74):
    full pivoting, column-major first maximum, count |u_kk| > threshold * max pivot."""
    a = np.array(a, dtype=np.float64)
    n = a.shape[0]
    maxpiv = 0.0
    for k in range(n):
        sub = np.abs(a[k:, k:])
        flat = int(np.argmax(sub.T.ravel()))  # column-major scan
        bj, bi = divmod(flat, n - k)
        big = sub[bi, bj]
        maxpiv = max(maxpiv, big)
        if big == 0.0:
            break
        a[[k, k + bi]] = a[[k + bi, k]]
        a[:, [k, k + bj]] = a[:, [k + bj, k]]
        a[k + 1:, k] /= a[k, k]
        a[k + 1:, k + 1:] -= np.outer(a[k + 1:, k], a[k, k + 1:])
    return int(np.sum(np.abs(np.diag(a)) > threshold * maxpiv))


def fit_var(coeffs, order):
    """fit_var (stochastic.cpp:30-107) restated in numpy: per coefficient the
    normal equations accumulated in (r, t) order, the rank rule of FullPivLU,
    phi by a dense solve, residuals, OLS standard errors, and the unstable count
    from the companion matrix eigenvalues (stochastic.cpp:19-27)."""
    c = np.asarray(coeffs, dtype=np.float64)
    r_len, t_len, d = c.shape
    if order == 0:
        mean = c.reshape(-1, d).sum(axis=0) / (r_len * t_len)
        res = (c - mean).reshape(-1, d)
        return dict(phi=np.zeros((0, d)), phi_se=np.zeros((0, d)), residuals=res, zeroed_count=0,
                    unstable_count=0, residual_mean_norm=float(np.linalg.norm(res.mean(axis=0))))
    rows = t_len - order
    X = np.stack([c[:, order - 1 - p:t_len - 1 - p, :] for p in range(order)], axis=-1)  # (r, rows, d, P)
    Y = c[:, order:, :]
    phi = np.zeros((order, d))
    se = np.zeros((order, d))
    res = np.empty((r_len * rows, d))
    zeroed = unstable = 0
    n_rows = r_len * rows
    for i in range(d):
        x = X[:, :, i, :].reshape(-1, order)
        y = Y[:, :, i].reshape(-1)
        a = np.zeros((order, order))
        b = np.zeros(order)
        for row in range(x.shape[0]):  # sequential accumulation like Eigen's a += x x^T
            a += np.outer(x[row], x[row])
            b += x[row] * y[row]
        degenerate = _fullpiv_rank(a) < order
        ph = np.zeros(order) if degenerate else np.linalg.solve(a, b)
        zeroed += degenerate
        phi[:, i] = ph
        e = y - x @ ph
        res[:, i] = e
        if not degenerate and n_rows > order:
            s2 = float(e @ e) / (n_rows - order)
            se[:, i] = np.sqrt(np.maximum(0.0, s2 * np.diag(np.linalg.inv(a))))
        comp = np.zeros((order, order))
        comp[0, :] = ph
        comp[1:, :-1] += np.eye(order - 1)
        rad = abs(ph[0]) if order == 1 else float(np.max(np.abs(np.linalg.eigvals(comp))))
        unstable += rad >= 1.0 - 1e-8
    return dict(phi=phi, phi_se=se, residuals=res, zeroed_count=int(zeroed), unstable_count=int(unstable),
                residual_mean_norm=float(np.linalg.norm(res.mean(axis=0))))


# ----------------------------------------------------------------------------
# train pipeline (pipeline.cpp:18-54) restated over the pieces above — the C1
# end-to-end checker (test infrastructure only)
# ----------------------------------------------------------------------------
def fit_trend(series, harmonics, period):
    """fit_trend(series, {}, TrendConfig) without forcing (trend.cpp:129-250):
    pooled mean over replicates, least squares by Householder QR (numpy's
    LAPACK QR for Eigen's HouseholderQR), sigma from the pooled residual plus
    the within-ensemble scatter, floored at 1e-12."""
    x = np.asarray(series, dtype=np.float64)
    if x.ndim == 2:
        x = x[None]
    r_len, t_len = x.shape[0], x.shape[1]
    points = x[0, 0].size
    y = x.reshape(r_len, t_len, points)
    ybar = np.zeros((t_len, points))
    for r in range(r_len):
        ybar += y[r]
    ybar /= r_len
    within = np.zeros(points)
    for r in range(r_len):
        d = y[r] - ybar
        within += (d * d).sum(axis=0)
    p = 1 + 2 * harmonics
    t = np.arange(1, t_len + 1)
    base = 2.0 * np.pi * (t % period) / period
    X = np.empty((t_len, p))
    X[:, 0] = 1.0
    for k in range(1, harmonics + 1):
        X[:, 2 * k - 1] = np.cos(base * k)
        X[:, 2 * k] = np.sin(base * k)
    q, rr = np.linalg.qr(X)
    beta = np.linalg.solve(rr, q.T @ ybar)
    resid = ybar - X @ beta
    rec = np.zeros((points, 5 + 2 * harmonics))
    rec[:, 0] = beta[0]
    for k in range(harmonics):
        rec[:, 4 + k] = beta[1 + 2 * k]
        rec[:, 4 + harmonics + k] = beta[2 + 2 * k]
    var = (r_len * (resid * resid).sum(axis=0) + within) / (r_len * t_len)
    rec[:, -1] = np.sqrt(np.maximum(var, 1e-12))
    return rec


def estimate_innovation_covariance(xi, variant="dp", tile=128):
    n, d = xi.shape
    u, v = np.empty((d, d)), np.empty((d, d))
    nug = C.c_double()
    st = CholStats()
    rc = lib().so_estimate_innovation_covariance(np.ascontiguousarray(xi), n, d, C.byref(config(variant, tile)), 1,
                                                 u, v, C.byref(nug), C.byref(st))
    if rc:
        raise RuntimeError("innovation covariance is not positive definite")
    return u, v, nug.value


def train(series, harmonics, period, var_order, band_limit, variant="dp", tile=128):
    """train(series, {}, TrainConfig) (pipeline.cpp:18-54): returns the model dict."""
    x = np.asarray(series, dtype=np.float64)
    if x.ndim == 3:
        x = x[None]
    r_len, t_len, nt, nphi = x.shape
    rec = fit_trend(x, harmonics, period)
    std = trend_apply("detrend", x.reshape(r_len, t_len, nt * nphi), rec, harmonics, period)
    plan = Plan(nt, nphi, band_limit)
    coeffs = plan.forward(std.reshape(-1, nt, nphi)).reshape(r_len, t_len, -1)
    vf = fit_var(coeffs, var_order)
    u, v, nug = estimate_innovation_covariance(vf["residuals"], variant, tile)
    recon = plan.inverse(coeffs.reshape(r_len * t_len, -1)).reshape(r_len, t_len, nt * nphi)
    e = std.reshape(r_len, t_len, -1) - recon
    v2 = (e * e).sum(axis=(0, 1)) / (r_len * t_len)
    return dict(records=rec, phi=vf["phi"], u_hat=u, v=v, nugget=nug, v2=v2, plan=plan, harmonics=harmonics,
                period=period, grid=(nt, nphi), band_limit=band_limit)


def emulate_model(model, t_out, seed, r_len=1, t_start=1, threads=1):
    """emulate(model, plan, {}, t_out, seed, r_len, threads, t_start) (stochastic.cpp:217-277)."""
    means = mean_table(model["records"], model["harmonics"], model["period"], t_out, t_start)
    sigma = np.ascontiguousarray(model["records"][:, -1])
    return emulate(model["plan"], model["v"], model["phi"] if model["phi"].shape[0] else None, means, sigma,
                   model["v2"], t_out, seed, r_len, threads)


def synth_training_series(n_theta, n_phi, band_limit, t_len, r_len, seed, period=12):
    """AR(1)-in-coefficients series with a seasonal cycle
    (acceptance_main.cpp:535-559): state = 0.55 state + 0.5/(1+l) N(0,1) per
    slot, inverse SHT, + 1.7 + 1.1 cos(2 pi (t+1)/period) + 0.05 N(0,1); one
    GaussianRng stream (slots, then points, per step)."""
    d = band_limit * band_limit
    points = n_theta * n_phi
    plan = Plan(n_theta, n_phi, band_limit)
    z = normals(seed, r_len * t_len * (d + points)).reshape(r_len, t_len, d + points)
    deg = np.floor(np.sqrt(np.arange(d))).astype(int)
    scale = 0.5 / (1.0 + deg)
    out = np.empty((r_len, t_len, n_theta, n_phi))
    for r in range(r_len):
        state = np.zeros(d)
        for t in range(t_len):
            for i in range(d):  # sequential like the reference (no vectorized FMA differences)
                state[i] = 0.55 * state[i] + scale[i] * z[r, t, i]
            synth = plan.inverse(state[None])[0].reshape(points)
            season = 1.1 * np.cos(2.0 * np.pi * (t + 1) / period)
            out[r, t] = (1.7 + season + synth + 0.05 * z[r, t, d:]).reshape(n_theta, n_phi)
    return out


def tile_norm_precisions(a, variant, tile_size, band_width_dp=1, tolerance=1e-8, hp_format="fp16"):
    """The tile-norm ("tile-centric") precision rule restated:
    off the DP band, tile (i, j) takes the lowest precision p the variant
    allows with u_p ||A_ij||_F <= tolerance ||A||_F / nt (so the storage
    rounding of all tiles sums to <= tolerance ||A||_F in Frobenius norm);
    packed i(i+1)/2 + j, 0/1/2 = dp/sp/hp."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    nt = (n + tile_size - 1) // tile_size
    total = np.linalg.norm(a)
    allowed = {"dp": [0], "dpsp": [1, 0], "dpsphp": [2, 1, 0], "dphp": [2, 0]}[variant]
    u = {0: 2.0 ** -53, 1: 2.0 ** -24, 2: 2.0 ** -11 if hp_format == "fp16" else 2.0 ** -8}
    out = np.zeros(nt * (nt + 1) // 2, dtype=np.uint8)
    for i in range(nt):
        for j in range(i + 1):
            if i - j < band_width_dp:
                continue
            t = np.linalg.norm(a[i * tile_size:(i + 1) * tile_size, j * tile_size:(j + 1) * tile_size])
            for p in allowed:
                if u[p] * t <= tolerance * total / nt:
                    out[i * (i + 1) // 2 + j] = p
                    break
    return out
