"""Python mirror of the reference's pybind11 module ``_sphemu``
(proj/bindings/module.cpp:183-246) over the B200 C-ABI (include/sphemu_gpu.h).

Same function names, argument names, defaults and error types as the
reference; every computation runs in lib/libsphemu_gpu.so on the GPU. There
is no CPU fallback: importing on a machine without the built library raises.
New keyword arguments are appended after the reference's and default to the
reference behaviour.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os

import numpy as np

__version__ = "0.1.0"  # proj/include/sphemu/version.hpp:4

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPHEMU_LIB") or os.path.join(_HERE, "lib", "libsphemu_gpu.so")

SPHEMU_OK, SPHEMU_ERR_INVALID_ARG, SPHEMU_ERR_NOT_SPD = 0, 1, 2
HOST, DEVICE = 0, 1
VARIANTS = {"dp": 0, "dpsp": 1, "dpsphp": 2, "dphp": 3}  # mpchol.cpp:47-53
_VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}


class NotPositiveDefiniteError(RuntimeError):
    """mpchol.hpp:122-130: carries the failing diagonal tile index."""

    def __init__(self, tile_index: int, what: str):
        super().__init__(what)
        self.tile_index = tile_index


class CholConfig(C.Structure):
    _fields_ = [("variant", C.c_int), ("tile_size", C.c_int), ("band_width_dp", C.c_int),
                ("sp_fraction", C.c_double), ("workers", C.c_int), ("hp_format", C.c_int),
                ("compute", C.c_int), ("lookahead", C.c_int), ("sp_compute", C.c_int)]


class CholStats(C.Structure):
    _fields_ = [("n", C.c_int), ("tile_size", C.c_int), ("n_tiles", C.c_int), ("workers", C.c_int),
                ("variant", C.c_int), ("tasks_potrf", C.c_int64), ("tasks_trsm", C.c_int64),
                ("tasks_syrk", C.c_int64), ("tasks_gemm", C.c_int64), ("tiles_dp", C.c_int64),
                ("tiles_sp", C.c_int64), ("tiles_hp", C.c_int64), ("bytes_dp", C.c_int64),
                ("bytes_sp", C.c_int64), ("bytes_hp", C.c_int64), ("demotions_sp", C.c_int64),
                ("demotions_hp", C.c_int64), ("half_saturations", C.c_int64),
                ("wall_seconds", C.c_double), ("device_ms", C.c_double), ("launches", C.c_int64)]

    def to_json(self) -> str:
        """FactorizationStats::to_json (mpchol.cpp:437-457): nlohmann's sorted
        keys, indent 2; GPU-only numbers under the new key "device"."""
        d = {
            "n": self.n, "tile_size": self.tile_size, "n_tiles": self.n_tiles,
            "workers": self.workers, "variant": _VARIANT_NAMES[self.variant],
            "tasks": {"potrf": self.tasks_potrf, "trsm": self.tasks_trsm,
                      "syrk": self.tasks_syrk, "gemm": self.tasks_gemm,
                      "total": self.tasks_potrf + self.tasks_trsm + self.tasks_syrk + self.tasks_gemm},
            "tiles": {"dp": self.tiles_dp, "sp": self.tiles_sp, "hp": self.tiles_hp},
            "bytes": {"dp": self.bytes_dp, "sp": self.bytes_sp, "hp": self.bytes_hp,
                      "total": self.bytes_dp + self.bytes_sp + self.bytes_hp},
            "conversions": {"to_sp": self.demotions_sp, "to_hp": self.demotions_hp,
                            "half_saturations": self.half_saturations},
            "wall_seconds": self.wall_seconds,
            "device": {"factor_ms": self.device_ms, "kernel_launches": self.launches},
        }
        return json.dumps(d, indent=2, sort_keys=True) + "\n"


_lib = None


def lib():
    """The native library; raises when it is not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback for the sphemu B200 path)")
        L = C.CDLL(LIB_PATH)
        vp, i64, dp = C.c_void_p, C.c_int64, C.POINTER(C.c_double)
        L.sphemu_gpu_last_error.restype = C.c_char_p
        L.sphemu_gpu_version.restype = C.c_char_p
        L.sphemu_gpu_launch_count.restype = i64
        L.sphemu_gpu_tiled_cholesky_dense.argtypes = [vp, C.c_int, C.c_int, C.POINTER(CholConfig), vp,
                                                      C.c_int, C.POINTER(CholStats), C.POINTER(C.c_int)]
        L.sphemu_gpu_chol_create.argtypes = [C.c_int, C.POINTER(CholConfig), C.POINTER(vp)]
        L.sphemu_gpu_chol_destroy.argtypes = [vp]
        L.sphemu_gpu_chol_load_dense.argtypes = [vp, vp, C.c_int, i64]
        L.sphemu_gpu_chol_generate_spd.argtypes = [vp, C.c_uint64]
        L.sphemu_gpu_chol_factor.argtypes = [vp]
        L.sphemu_gpu_chol_wait.argtypes = [vp, C.POINTER(CholStats), C.POINTER(C.c_int)]
        L.sphemu_gpu_chol_store_dense.argtypes = [vp, vp, C.c_int, i64]
        L.sphemu_gpu_chol_residual.argtypes = [vp, vp, C.c_int, i64, dp]
        L.sphemu_gpu_chol_flops.argtypes = [vp, dp, dp, dp]
        L.sphemu_gpu_chol_stream.argtypes = [vp]
        L.sphemu_gpu_chol_stream.restype = vp
        L.sphemu_gpu_assign_precisions.argtypes = [C.c_int, C.POINTER(CholConfig), vp]
        L.sphemu_gpu_chol_config_validate.argtypes = [C.POINTER(CholConfig)]
        L.sphemu_gpu_sht_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_size_t, C.POINTER(vp)]
        L.sphemu_gpu_sht_destroy.argtypes = [vp]
        L.sphemu_gpu_sht_forward.argtypes = [vp, vp, C.c_int, i64, vp, C.c_int]
        L.sphemu_gpu_sht_inverse.argtypes = [vp, vp, C.c_int, i64, vp, C.c_int]
        L.sphemu_gpu_sht_stream.argtypes = [vp]
        L.sphemu_gpu_synth_bandlimited.argtypes = [vp, C.c_int, i64, C.c_int, C.c_int, C.c_int, vp,
                                                   C.c_int]
        L.sphemu_gpu_sht_stream.restype = vp
        L.sphemu_gpu_sht_plan_seconds.argtypes = [vp]
        L.sphemu_gpu_sht_plan_seconds.restype = C.c_double
        L.sphemu_gpu_nccl_unique_id.argtypes = [vp]
        L.sphemu_gpu_wigner_d_half_pi.argtypes = [C.c_int, C.c_size_t, i64, vp, vp, vp, vp,
                                                  C.POINTER(C.c_int)]
        L.sphemu_gpu_chol_create_dist.argtypes = [C.c_int, C.POINTER(CholConfig), C.c_int, C.c_int, C.c_int, vp,
                                                  C.POINTER(vp)]
        L.sphemu_gpu_chol_set_profiling.argtypes = [vp, C.c_int]
        L.sphemu_gpu_chol_phase_times.argtypes = [vp, vp, vp, C.c_int]
        L.sphemu_gpu_chol_update_flops.argtypes = [vp, dp, dp, dp]
        L.sphemu_gpu_chol_timeline.argtypes = [vp, vp, vp, vp, vp, C.c_int, C.POINTER(C.c_int)]
        L.sphemu_gpu_chol_residual_probe_spd.argtypes = [vp, C.c_uint64, C.c_int, dp]
        L.sphemu_gpu_emulate.argtypes = [vp, vp, C.c_int, vp, C.c_int, vp, vp, vp, C.c_int, C.c_uint64,
                                         C.c_int, C.c_int, vp]
        L.sphemu_gpu_emulate_range.argtypes = [vp, vp, C.c_int, vp, C.c_int, vp, vp, vp, C.c_int, C.c_uint64,
                                               C.c_int, C.c_int, C.c_int, vp]
        L.sphemu_gpu_estimate_innovation_covariance.argtypes = [
            vp, C.c_int, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(CholConfig), vp, C.c_int, vp, C.c_int,
            dp, C.POINTER(CholStats)]
        trend = [vp, C.c_int, C.c_int, C.c_int, vp, i64, C.c_int, C.c_int, vp, i64, vp, i64, i64, vp, C.c_int]
        L.sphemu_gpu_mean_table.argtypes = [vp, i64, C.c_int, C.c_int, vp, i64, vp, i64, C.c_int, i64, vp,
                                            C.c_int]
        L.sphemu_gpu_emulate_trend.argtypes = [vp, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, vp, i64, vp,
                                               i64, i64, vp, C.c_int, C.c_uint64, C.c_int, C.c_int, vp]
        L.sphemu_gpu_fit_var.argtypes = [vp, C.c_int, C.c_int, C.c_int, i64, C.c_int, vp, vp, vp, C.c_int,
                                         C.POINTER(i64), C.POINTER(i64), dp]
        L.sphemu_gpu_chol_trmm.argtypes = [vp, vp, C.c_int, i64, vp, C.c_int]
        L.sphemu_gpu_chol_create_map.argtypes = [C.c_int, C.POINTER(CholConfig), vp, C.POINTER(vp)]
        L.sphemu_gpu_tile_norm_precisions.argtypes = [vp, C.c_int, i64, C.c_int, C.POINTER(CholConfig), C.c_double,
                                                      vp]
        L.sphemu_gpu_fit_trend.argtypes = [vp, C.c_int, C.c_int, C.c_int, i64, C.c_int, C.c_int, vp, C.c_int]
        L.sphemu_gpu_noise_field.argtypes = [vp, vp, C.c_int, i64, i64, vp, C.c_int]
        L.sphemu_gpu_innovation_factor.argtypes = [vp, C.c_int, i64, C.c_int, C.c_int, C.c_int, C.c_int,
                                                   C.POINTER(CholConfig), vp, C.c_int, dp, C.POINTER(CholStats),
                                                   C.POINTER(vp)]
        L.sphemu_gpu_chol_load_factor.argtypes = [vp, vp, C.c_int, i64]
        L.sphemu_gpu_emulate_chol_trend.argtypes = [vp, vp, vp, C.c_int, vp, C.c_int, C.c_int, vp, i64, vp, i64,
                                                    i64, vp, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, vp,
                                                    C.c_int]
        L.sphemu_gpu_emulate_chol.argtypes = [vp, vp, vp, C.c_int, vp, vp, vp, C.c_int, C.c_uint64, C.c_int,
                                              C.c_int, C.c_int, vp, C.c_int]
        L.sphemu_gpu_detrend.argtypes = trend
        L.sphemu_gpu_retrend.argtypes = trend
        _lib = L
    return _lib


def _check(rc: int, failed_tile: int = -1):
    if rc == SPHEMU_OK:
        return
    msg = lib().sphemu_gpu_last_error().decode()
    if rc == SPHEMU_ERR_INVALID_ARG:
        raise ValueError(msg)
    if rc == SPHEMU_ERR_NOT_SPD:
        raise NotPositiveDefiniteError(failed_tile, msg)
    raise RuntimeError(msg)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


# SP-class arithmetic (tensor mode): "fp16x3" row-scaled fp16 hi+lo on kind::f16
# (default), "tf32x3" on kind::tf32, "fp64" the oracle's FP64 arithmetic on
# the SP tiles (DMMA; exact parity with mpchol.cpp at ~6x the SP-class time).
SP_COMPUTE = {"fp16x3": 0, "tf32x3": 1, "fp64": 2}


def make_config(variant="dp", tile_size=128, workers=1, band_width_dp=1, sp_fraction=0.05,
                hp_format="fp16", compute="tensor", lookahead=0, sp_compute="fp16x3") -> CholConfig:
    if variant not in VARIANTS:
        raise ValueError(f"unknown precision variant: {variant}")  # mpchol.cpp:52
    if hp_format not in ("fp16", "bf16"):
        raise ValueError(f"unknown half-precision format: {hp_format}")
    if compute not in ("tensor", "fp64"):
        raise ValueError(f"unknown compute mode: {compute}")
    if sp_compute not in SP_COMPUTE:
        raise ValueError(f"unknown single-precision compute: {sp_compute}")
    return CholConfig(VARIANTS[variant], tile_size, band_width_dp, sp_fraction, workers,
                      1 if hp_format == "bf16" else 0, 0 if compute == "tensor" else 1, lookahead,
                      SP_COMPUTE[sp_compute])


# ---------------------------------------------------------------------------
# module.cpp:209-214 tiled_cholesky / make_spd_matrix
# ---------------------------------------------------------------------------
def tile_norm_precisions(a, variant="dpsphp", tile_size=128, band_width_dp=1, tolerance=1e-8, hp_format="fp16"):
    """Tile-norm precision map (sphemu_gpu_tile_norm_precisions): off the DP
    band, each tile takes the lowest precision the variant allows with
    u_p ||A_ij||_F <= tolerance ||A||_F / n_tiles."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    nt = (n + tile_size - 1) // tile_size
    cfg = make_config(variant, tile_size, 1, band_width_dp, 0.05, hp_format)
    out = np.empty(nt * (nt + 1) // 2, dtype=np.uint8)
    _check(lib().sphemu_gpu_tile_norm_precisions(_ptr(a), HOST, n, n, C.byref(cfg), C.c_double(tolerance), _ptr(out)))
    return out


def tiled_cholesky(a, variant="dp", tile_size=128, workers=1, band_width_dp=1, sp_fraction=0.05,
                   hp_format="fp16", compute="tensor", lookahead=1, sp_compute="fp16x3", precision_policy="band",
                   norm_tolerance=1e-8):
    """Tiled Cholesky factorization; returns (lower_factor, stats_json).
    precision_policy="norm" replaces the band rule by the tile-norm map
    (tile_norm_precisions) at norm_tolerance."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("expected a square matrix")
    n = a.shape[0]
    if precision_policy not in ("band", "norm"):
        raise ValueError(f"unknown precision policy: {precision_policy}")
    if precision_policy == "norm":
        pm = tile_norm_precisions(a, variant, tile_size, band_width_dp, norm_tolerance, hp_format)
        h = Cholesky(n, variant, tile_size, workers, band_width_dp, sp_fraction, hp_format, compute, lookahead,
                     sp_compute, precision_map=pm)
        h.load(a)
        h.factor()
        st = h.wait()
        return h.factor_dense(), st.to_json()
    cfg = make_config(variant, tile_size, workers, band_width_dp, sp_fraction, hp_format, compute, lookahead,
                      sp_compute)
    out = np.empty_like(a)
    st = CholStats()
    failed = C.c_int(-1)
    rc = lib().sphemu_gpu_tiled_cholesky_dense(_ptr(a), HOST, n, C.byref(cfg), _ptr(out), HOST,
                                               C.byref(st), C.byref(failed))
    _check(rc, failed.value)
    return out, st.to_json()


def make_spd_matrix(n, seed=1):
    """make_spd_test_matrix (mpchol.cpp:419-435), generated on the device."""
    if n < 1:
        raise ValueError("matrix size must be positive")
    h = Cholesky(n, variant="dp", tile_size=min(1024, max(64, n)), compute="fp64")
    h.generate_spd(seed)
    lower = h.factor_dense_unfactored()
    return lower + np.tril(lower, -1).T


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (create on rank 0, share with the others)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().sphemu_gpu_nccl_unique_id(C.byref(buf)))
    return bytes(buf)


class Cholesky:
    """Device-resident factorization (TiledMatrix + tiled_cholesky).

    dist=(P, Q, rank, uid) distributes the tiles 2D block-cyclically over a
    P x Q grid of GPUs (one process per GPU, device already selected); every
    method is then collective, and factor_dense() returns the gathered factor
    on rank 0 (None elsewhere)."""

    def __init__(self, n, variant="dp", tile_size=128, workers=1, band_width_dp=1, sp_fraction=0.05,
                 hp_format="fp16", compute="tensor", lookahead=1, sp_compute="fp16x3", dist=None,
                 precision_map=None):
        self.n = n
        self.cfg = make_config(variant, tile_size, workers, band_width_dp, sp_fraction, hp_format,
                               compute, lookahead, sp_compute)
        h = C.c_void_p()
        self.rank = 0
        self.dist = dist
        if precision_map is not None:
            if dist is not None:
                raise ValueError("explicit precision maps are single-GPU")
            pm = np.ascontiguousarray(precision_map, dtype=np.uint8)
            _check(lib().sphemu_gpu_chol_create_map(n, C.byref(self.cfg), _ptr(pm), C.byref(h)))
        elif dist is None:
            _check(lib().sphemu_gpu_chol_create(n, C.byref(self.cfg), C.byref(h)))
        else:
            P, Q, rank, uid = dist
            self.rank = rank
            ub = (C.c_uint8 * 128).from_buffer_copy(uid)
            _check(lib().sphemu_gpu_chol_create_dist(n, C.byref(self.cfg), P, Q, rank, C.byref(ub), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter shutdown
            lib().sphemu_gpu_chol_destroy(self.h)
            self.h = None

    def generate_spd(self, seed=1, rho=None):
        """make_spd_test_matrix(n, seed) into the tiles; rho (0 < rho < 1)
        replaces the reference's 0.9 decay (non-decaying tiles as rho -> 1)."""
        if rho is None:
            _check(lib().sphemu_gpu_chol_generate_spd(self.h, seed))
        else:
            _check(lib().sphemu_gpu_chol_generate_spd_decay(self.h, C.c_uint64(seed), C.c_double(rho)))

    def load(self, a, where=HOST, lda=None):
        if where == HOST:
            a = np.ascontiguousarray(a, dtype=np.float64)
            _check(lib().sphemu_gpu_chol_load_dense(self.h, _ptr(a), HOST, a.shape[1]))
        else:  # device pointer (int) with row stride
            _check(lib().sphemu_gpu_chol_load_dense(self.h, C.c_void_p(a), DEVICE, lda or self.n))

    def factor(self):
        _check(lib().sphemu_gpu_chol_factor(self.h))

    def wait(self):
        st = CholStats()
        failed = C.c_int(-1)
        rc = lib().sphemu_gpu_chol_wait(self.h, C.byref(st), C.byref(failed))
        _check(rc, failed.value)
        return st

    def factor_dense(self):
        out = np.empty((self.n, self.n))
        _check(lib().sphemu_gpu_chol_store_dense(self.h, _ptr(out), HOST, self.n))
        return out if self.rank == 0 else None

    factor_dense_unfactored = factor_dense  # the stored tiles, before or after factor()

    def store(self, dev_ptr, ld=None):
        _check(lib().sphemu_gpu_chol_store_dense(self.h, C.c_void_p(dev_ptr or 0), DEVICE, ld or self.n))

    def residual(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = C.c_double()
        _check(lib().sphemu_gpu_chol_residual(self.h, _ptr(a), HOST, a.shape[1], C.byref(out)))
        return out.value

    def flops(self):
        f = [C.c_double() for _ in range(3)]
        _check(lib().sphemu_gpu_chol_flops(self.h, *[C.byref(x) for x in f]))
        return {"dp": f[0].value, "sp": f[1].value, "hp": f[2].value}

    @property
    def stream(self):
        return lib().sphemu_gpu_chol_stream(self.h)

    PHASES = ("potrf", "panel", "update_dp", "update_sp", "update_hp", "load", "exchange")

    def set_profiling(self, on=True, phases=None):
        """Record phase times; phases (names of PHASES) limits which."""
        v = 1 if on else 0
        if on and phases is not None:
            v = 0x100 | sum(1 << self.PHASES.index(p) for p in phases)
        _check(lib().sphemu_gpu_chol_set_profiling(self.h, v))

    def phase_times(self, reset=False):
        ms = np.zeros(len(self.PHASES))
        cnt = np.zeros(len(self.PHASES), dtype=np.int64)
        _check(lib().sphemu_gpu_chol_phase_times(self.h, _ptr(ms), _ptr(cnt), 1 if reset else 0))
        return {p: {"ms": float(ms[i]), "launches": int(cnt[i])} for i, p in enumerate(self.PHASES)}

    def timeline(self, cap=100000):
        """[(phase, stream, t0_ms, t1_ms)] of the last profiled factorization."""
        ph = np.zeros(cap, dtype=np.int32)
        st = np.zeros(cap, dtype=np.int32)
        t0 = np.zeros(cap)
        t1 = np.zeros(cap)
        n = C.c_int()
        _check(lib().sphemu_gpu_chol_timeline(self.h, _ptr(ph), _ptr(st), _ptr(t0), _ptr(t1), cap, C.byref(n)))
        k = min(n.value, cap)
        return [(self.PHASES[ph[i]], int(st[i]), float(t0[i]), float(t1[i])) for i in range(k)]

    def reset_phase_times(self):
        self.phase_times(reset=True)

    def class_update_flops(self):
        f = [C.c_double() for _ in range(3)]
        _check(lib().sphemu_gpu_chol_update_flops(self.h, *[C.byref(x) for x in f]))
        return {"dp": f[0].value, "sp": f[1].value, "hp": f[2].value}

    def residual_probe(self, seed=1, n_vec=2, rho=None):
        out = C.c_double()
        if rho is None:
            _check(lib().sphemu_gpu_chol_residual_probe_spd(self.h, seed, n_vec, C.byref(out)))
        else:
            _check(lib().sphemu_gpu_chol_residual_probe_spd_decay(self.h, C.c_uint64(seed), C.c_double(rho), n_vec,
                                                                   C.byref(out)))
        return out.value

    def trmm(self, eta):
        """xi = eta L^T (row per snapshot) over the stored tiles: the emulation
        generator's innovation product alone (sphemu_gpu_chol_trmm)."""
        eta = np.ascontiguousarray(eta, dtype=np.float64)
        out = np.empty((eta.shape[0], self.n))
        _check(lib().sphemu_gpu_chol_trmm(self.h, _ptr(eta), HOST, eta.shape[0], _ptr(out), HOST))
        return out

    def emulate(self, plan, phi, means, sigma, v2, t_out, seed=1, r_len=1, rng="philox", r_begin=0, out_ptr=None):
        """emulate (stochastic.cpp:217-277) with V = this handle's tiled factor
        (sphemu_gpu_emulate_chol); distributed handles return this rank's
        contiguous block of the replicates."""
        d = self.n
        phi = np.zeros((0, d)) if phi is None else np.ascontiguousarray(phi, dtype=np.float64).reshape(-1, d)
        phi_a = phi if phi.shape[0] else np.zeros((1, d))
        means = np.ascontiguousarray(means, dtype=np.float64)
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        v2 = np.ascontiguousarray(v2, dtype=np.float64)
        world = 1 if self.dist is None else self.dist[0] * self.dist[1]
        rank = self.rank
        lo = r_begin + (r_len * rank) // world
        hi = r_begin + (r_len * (rank + 1)) // world
        mode = {"reference": 0, "philox": 1}[rng]
        if out_ptr is not None:  # device buffer of (hi - lo, t_out, n_theta, n_phi) doubles
            _check(lib().sphemu_gpu_emulate_chol(self.h, plan.h, _ptr(phi_a), phi.shape[0], _ptr(means),
                                                 _ptr(sigma), _ptr(v2), t_out, seed, r_begin, r_len, mode,
                                                 C.c_void_p(out_ptr), DEVICE))
            return hi - lo
        out = np.empty((hi - lo, t_out, plan.n_theta, plan.n_phi))
        _check(lib().sphemu_gpu_emulate_chol(self.h, plan.h, _ptr(phi_a), phi.shape[0], _ptr(means), _ptr(sigma),
                                             _ptr(v2), t_out, seed, r_begin, r_len, mode, _ptr(out), HOST))
        return out


def emulate(plan, v, phi, means, sigma, v2, t_out, seed=1, r_len=1, rng="reference", r_begin=0):
    """emulate (stochastic.cpp:217-277) with the trend evaluated by the caller
    (means: t_out x points, sigma/v2: points). rng="reference" reproduces the
    reference's serial mt19937_64 stream; "philox" draws on the device."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    d = v.shape[0]
    phi = np.zeros((0, d)) if phi is None else np.ascontiguousarray(phi, dtype=np.float64).reshape(-1, d)
    phi_a = phi if phi.shape[0] else np.zeros((1, d))
    means = np.ascontiguousarray(means, dtype=np.float64)
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    v2 = np.ascontiguousarray(v2, dtype=np.float64)
    out = np.empty((r_len, t_out, plan.n_theta, plan.n_phi))
    mode = {"reference": 0, "philox": 1}[rng]
    if r_begin:
        _check(lib().sphemu_gpu_emulate_range(plan.h, _ptr(v), d, _ptr(phi_a), phi.shape[0], _ptr(means),
                                              _ptr(sigma), _ptr(v2), t_out, seed, r_begin, r_len, mode, _ptr(out)))
    else:
        _check(lib().sphemu_gpu_emulate(plan.h, _ptr(v), d, _ptr(phi_a), phi.shape[0], _ptr(means), _ptr(sigma),
                                        _ptr(v2), t_out, seed, r_len, mode, _ptr(out)))
    return out


def estimate_innovation_covariance(residuals, r_len, t_len, order, variant="dp", tile_size=128, workers=1,
                                   band_width_dp=1, sp_fraction=0.05, hp_format="fp16", compute="tensor",
                                   lookahead=1, sp_compute="fp64"):
    """estimate_innovation_covariance (stochastic.cpp:109-172) on the device:
    returns (u_hat, v, nugget, stats_json) like InnovationModel
    (stochastic.hpp:36-42); residuals is the (r_len*(t_len-order)) x d matrix.

    The nugget is a discrete decision taken on the factorization's success,
    so the SP class defaults to its FP64 arithmetic here (the oracle's): the
    fp16x3 tensor form may need a larger nugget on rank-deficient input."""
    xi = np.ascontiguousarray(residuals, dtype=np.float64)
    if xi.ndim != 2:
        raise ValueError("residuals must be a 2-D array")
    d = xi.shape[1]
    cfg = make_config(variant, tile_size, workers, band_width_dp, sp_fraction, hp_format, compute, lookahead,
                      sp_compute)
    u = np.empty((d, d))
    v = np.empty((d, d))
    nug = C.c_double()
    st = CholStats()
    _check(lib().sphemu_gpu_estimate_innovation_covariance(_ptr(xi), HOST, xi.shape[0], d, r_len, t_len, order,
                                                           C.byref(cfg), _ptr(u), HOST, _ptr(v), HOST,
                                                           C.byref(nug), C.byref(st)))
    return u, v, nug.value, st.to_json()


def assign_precisions(n_tiles, variant="dp", band_width_dp=1, sp_fraction=0.05):
    """assign_precisions (mpchol.cpp:67-93): packed i(i+1)/2 + j, 0/1/2 = dp/sp/hp."""
    cfg = make_config(variant, 128, 1, band_width_dp, sp_fraction)
    out = np.empty(n_tiles * (n_tiles + 1) // 2, dtype=np.uint8)
    _check(lib().sphemu_gpu_assign_precisions(n_tiles, C.byref(cfg), _ptr(out)))
    return out


# ---------------------------------------------------------------------------
# module.cpp:194-198 forward_sht / inverse_sht (+ batch plans)
# ---------------------------------------------------------------------------
def _out(out, shape):
    if out is None:
        return np.empty(shape)
    if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != int(np.prod(shape)):
        raise ValueError(f"out must be a C-contiguous float64 array of {int(np.prod(shape))} values")
    return out


class ShtPlan:
    """build_plan(GridSpec{n_theta, n_phi}, band_limit) on the device."""

    def __init__(self, n_theta, n_phi, band_limit, wigner_cap_bytes=0):
        self.n_theta, self.n_phi, self.band_limit = n_theta, n_phi, band_limit
        h = C.c_void_p()
        _check(lib().sphemu_gpu_sht_create(n_theta, n_phi, band_limit, wigner_cap_bytes, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().sphemu_gpu_sht_destroy(self.h)
            self.h = None

    @property
    def plan_seconds(self):
        return lib().sphemu_gpu_sht_plan_seconds(self.h)

    @property
    def stream(self):
        return lib().sphemu_gpu_sht_stream(self.h)

    def forward(self, fields, out=None):
        """forward_sht_batch; out (optional): a C-contiguous float64 array of
        (n, L^2) values written in place (no intermediate copy)."""
        f = np.ascontiguousarray(fields, dtype=np.float64).reshape(-1, self.n_theta * self.n_phi)
        out = _out(out, (f.shape[0], self.band_limit ** 2))
        _check(lib().sphemu_gpu_sht_forward(self.h, _ptr(f), HOST, f.shape[0], _ptr(out), HOST))
        return out

    def inverse(self, coeffs, out=None):
        """inverse_sht_batch; out (optional): (n, n_theta, n_phi) float64, written in place."""
        c = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1, self.band_limit ** 2)
        out = _out(out, (c.shape[0], self.n_theta, self.n_phi))
        _check(lib().sphemu_gpu_sht_inverse(self.h, _ptr(c), HOST, c.shape[0], _ptr(out), HOST))
        return out

    def forward_device(self, fields_ptr, n, coeffs_ptr):
        _check(lib().sphemu_gpu_sht_forward(self.h, C.c_void_p(fields_ptr), DEVICE, n,
                                            C.c_void_p(coeffs_ptr), DEVICE))

    def inverse_device(self, coeffs_ptr, n, fields_ptr):
        _check(lib().sphemu_gpu_sht_inverse(self.h, C.c_void_p(coeffs_ptr), DEVICE, n,
                                            C.c_void_p(fields_ptr), DEVICE))


def _band_limit_of_coeffs(count):
    big_l = int(round(math.sqrt(count)))
    if big_l * big_l != count:
        raise ValueError("coefficient length must be a perfect square")
    return big_l


def max_band_limit(n_theta, n_phi):
    """GridSpec::max_band_limit (grid.cpp:27-29)."""
    if n_theta < 2:
        raise ValueError("grid needs at least two latitude rings")
    if n_phi < 1:
        raise ValueError("grid needs at least one longitude point")
    return min(n_theta - 1, (n_phi + 1) // 2)


def forward_sht(field, band_limit=0):
    """Analyze a (theta, phi) field into packed real harmonic coefficients."""
    f = np.ascontiguousarray(field, dtype=np.float64)
    if f.ndim != 2:
        raise ValueError("expected a (theta, phi) array")
    if band_limit == 0:
        band_limit = max_band_limit(*f.shape)
    return ShtPlan(f.shape[0], f.shape[1], band_limit).forward(f)[0]


def inverse_sht(coeffs, n_theta=0, n_phi=0):
    """Synthesize packed coefficients on a grid (tight grid by default)."""
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    if c.ndim != 1:
        raise ValueError("expected a flat coefficient array")
    big_l = _band_limit_of_coeffs(c.shape[0])
    if n_theta <= 0:
        n_theta, n_phi = big_l + 1, 2 * big_l  # GridSpec::from_band_limit
    if big_l > max_band_limit(n_theta, n_phi):
        return synth_bandlimited(c, n_theta, n_phi)  # module.cpp:92-94
    return ShtPlan(n_theta, n_phi, big_l).inverse(c)[0]


def synth_bandlimited(coeffs, n_theta, n_phi):
    """synth_bandlimited (sht.cpp:435-466): direct synthesis on any grid.

    coeffs is (L^2,) or (n, L^2); the result is (n_theta, n_phi) or
    (n, n_theta, n_phi).
    """
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    single = c.ndim == 1
    c2 = c.reshape(1, -1) if single else c
    if c2.ndim != 2:
        raise ValueError("expected (L^2,) or (n, L^2) coefficients")
    big_l = _band_limit_of_coeffs(c2.shape[1])
    max_band_limit(n_theta, n_phi)  # grid validation (grid.cpp:27-29)
    out = np.empty((c2.shape[0], n_theta, n_phi), dtype=np.float64)
    _check(lib().sphemu_gpu_synth_bandlimited(_ptr(c2), HOST, c2.shape[0], big_l, n_theta, n_phi,
                                              _ptr(out), HOST))
    return out[0] if single else out


def wigner_d_half_pi(l, m2, m):
    """wigner_d_half_pi(l, m2, m) (bindings/module.cpp:201-207): d^l_{m2,m}(pi/2)
    from the tables of build_wigner_tables(l + 1) (wigner.cpp:49-150), built on
    the device. Scalars give a float; equal-shape integer arrays give an array
    (one table build, band limit max(l) + 1)."""
    ls, m2s, ms = (np.ascontiguousarray(np.asarray(x), dtype=np.int32) for x in (l, m2, m))
    if not (ls.shape == m2s.shape == ms.shape):
        raise ValueError("l, m2 and m must have the same shape")
    if ls.size == 0:
        return np.empty(ls.shape, dtype=np.float64)
    out = np.empty(ls.shape, dtype=np.float64)
    _check(lib().sphemu_gpu_wigner_d_half_pi(int(ls.max()) + 1, 0, ls.size, _ptr(ls), _ptr(m2s), _ptr(ms),
                                             _ptr(out), None))
    return float(out) if out.ndim == 0 else out


def resolution_summary(band_limit):
    """resolution_summary (grid.cpp:40-48)."""
    if band_limit < 2:
        raise ValueError("band limit must be at least 2")
    return {"band_limit": band_limit, "degrees_per_cell": 180.0 / band_limit,
            "km_per_cell": 180.0 * 111.2 / band_limit,
            "grid_points": (band_limit - 1) * (2 * band_limit)}


class ForcingTrajectory:
    """ForcingTrajectory (trend.hpp:24-35): x[k] is year k+1, history[k] is
    year -k (newest first). Empty (both None) = no forcing terms."""

    def __init__(self, x=None, history=None):
        self.x = np.ascontiguousarray(np.zeros(0) if x is None else x, dtype=np.float64).ravel()
        self.history = np.ascontiguousarray(np.zeros(0) if history is None else history, dtype=np.float64).ravel()

    def empty(self) -> bool:
        return self.x.size == 0 and self.history.size == 0


def _forcing_args(forcing):
    f = forcing if isinstance(forcing, ForcingTrajectory) else ForcingTrajectory(
        *(forcing if forcing is not None else (None, None)))
    return f, [_ptr(f.x) if f.x.size else None, f.x.size, _ptr(f.history) if f.history.size else None,
               f.history.size]


def _records(records, harmonics):
    rec = np.ascontiguousarray(records, dtype=np.float64)
    stride = 5 + 2 * harmonics
    if rec.size % stride:
        raise ValueError(f"records must hold (5 + 2*harmonics) = {stride} values per location")
    return rec, rec.size // stride


def mean_table(records, harmonics, period, t_len, t_start=1, forcing=None):
    """mean_table (trend.cpp:252-287) on the device: (t_len, points) means of
    the TrendModel records (points x (5 + 2*harmonics)) for steps
    t_start..t_start+t_len-1. forcing: ForcingTrajectory or (x, history)."""
    rec, points = _records(records, harmonics)
    f, fa = _forcing_args(forcing)
    out = np.empty((t_len, points))
    _check(lib().sphemu_gpu_mean_table(_ptr(rec), points, harmonics, period, *fa, t_len, t_start, _ptr(out), HOST))
    return out


def _trend_apply(fn, series, records, harmonics, period, forcing, t_start):
    rec, points = _records(records, harmonics)
    f, fa = _forcing_args(forcing)
    x = np.ascontiguousarray(series, dtype=np.float64)
    if x.ndim == 2:
        x = x[None]
    r_len, t_len = x.shape[0], x.shape[1]
    if x.size != r_len * t_len * points:
        raise ValueError("series grid differs from model")
    out = np.empty(x.shape)
    _check(fn(_ptr(x), HOST, r_len, t_len, _ptr(rec), points, harmonics, period, *fa, t_start, _ptr(out), HOST))
    return out.reshape(np.shape(series))


def detrend(series, records, harmonics, period, forcing=None, t_start=1):
    """detrend (trend.cpp:289-305): (y - m_t) / sigma over a (r, t, ...)
    series whose trailing axes hold the model's points."""
    return _trend_apply(lib().sphemu_gpu_detrend, series, records, harmonics, period, forcing, t_start)


def retrend(standardized, records, harmonics, period, forcing=None, t_start=1):
    """retrend (trend.cpp:307-324): m_t + sigma * z."""
    return _trend_apply(lib().sphemu_gpu_retrend, standardized, records, harmonics, period, forcing, t_start)


def emulate_model(plan, v, phi, records, harmonics, period, v2, t_out, seed=1, r_len=1, t_start=1, forcing=None,
                  rng="reference"):
    """emulate(model, plan, forcing, t_out, seed, r_len, threads, t_start)
    (stochastic.cpp:217-277) with the model's trend as TrendModel records
    (points x (5 + 2*harmonics)): the mean table and sigma are evaluated on
    the device (trend.cu) instead of by the caller."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    d = v.shape[0]
    phi = np.zeros((0, d)) if phi is None else np.ascontiguousarray(phi, dtype=np.float64).reshape(-1, d)
    phi_a = phi if phi.shape[0] else np.zeros((1, d))
    rec, points = _records(records, harmonics)
    if points != plan.n_theta * plan.n_phi:
        raise ValueError("trend model grid differs from the transform plan")
    f, fa = _forcing_args(forcing)
    v2 = np.ascontiguousarray(v2, dtype=np.float64)
    out = np.empty((r_len, t_out, plan.n_theta, plan.n_phi))
    _check(lib().sphemu_gpu_emulate_trend(plan.h, _ptr(v), d, _ptr(phi_a), phi.shape[0], _ptr(rec), harmonics,
                                          period, *fa, t_start, _ptr(v2), t_out, seed, r_len,
                                          {"reference": 0, "philox": 1}[rng], _ptr(out)))
    return out


class VarFit:
    """VarFit (stochastic.hpp:29-37): phi / phi_se are order x d (row p-1 is
    lag p), residuals (r_len * (t_len - order)) x d, replicate-major."""

    def __init__(self, phi, phi_se, residuals, zeroed_count, unstable_count, residual_mean_norm):
        self.phi, self.phi_se, self.residuals = phi, phi_se, residuals
        self.zeroed_count, self.unstable_count = zeroed_count, unstable_count
        self.residual_mean_norm = residual_mean_norm


def fit_var(coeffs, order):
    """fit_var (stochastic.cpp:30-107) on the device: coeffs is the
    (r_len, t_len, d) packed coefficient series (CoeffSeries, sht.hpp:45-69)."""
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    if c.ndim == 2:
        c = c[None]
    r_len, t_len, d = c.shape
    rows = r_len * (t_len - order) if order > 0 else r_len * t_len
    phi = np.zeros((max(order, 0), d))
    se = np.zeros((max(order, 0), d))
    res = np.empty((max(rows, 0), d))
    zc, uc, nrm = C.c_int64(), C.c_int64(), C.c_double()
    _check(lib().sphemu_gpu_fit_var(_ptr(c), HOST, r_len, t_len, d, order, _ptr(phi) if order > 0 else None,
                                    _ptr(se) if order > 0 else None, _ptr(res), HOST, C.byref(zc), C.byref(uc),
                                    C.byref(nrm)))
    return VarFit(phi, se, res, zc.value, uc.value, nrm.value)
