"""The Python Emulator drop-in (bindings/module.cpp:140-179, 232-243) and the
model-bundle / field-series file formats it reads and writes, on the B200 path.

train (pipeline.cpp:18-54) runs every stage on the device through the C-ABI,
keeping the series in HBM between them: fit_trend + detrend (trend.cu),
forward SHT (sht.cu), fit_var (var.cu), the innovation covariance + nugget
loop with the factor kept as a device-resident tiled handle (chol.cu), the
inverse SHT and the noise field. emulate (stochastic.cpp:217-277) draws from
that handle (sphemu_gpu_emulate_chol_trend: xi = V eta as a TRMM over the
stored tiles, no dense V). save / load write and read the reference's
little-endian bundle files (trend.bin TRND, var.bin VARM, ucov.bin UCOV,
noise.bin NOIS, provenance.json; pipeline.cpp:56-97, stochastic.cpp:279-350,
trend.cpp:326-354) and read_sphf / write_sphf the SPHF series (grid.cpp:69-106).
"""
import ctypes as C
import json
import os
import struct

import numpy as np

from . import _sphemu as S

VERSION = "0.1.0"
_SPHF_VERSION = 1
_VARIANTS = ["dp", "dpsp", "dpsphp", "dphp"]


# ---------------------------------------------------------------------------
# little-endian binary helpers (io_util.hpp)
# ---------------------------------------------------------------------------
class _Writer:
    def __init__(self, path):
        self.f = open(path, "wb")

    def magic(self, m):
        self.f.write(m.encode())

    def u32(self, v):
        self.f.write(struct.pack("<I", int(v)))

    def f64(self, v):
        self.f.write(struct.pack("<d", float(v)))

    def f64s(self, a):
        self.f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())

    def close(self):
        self.f.close()


class _Reader:
    def __init__(self, path):
        self.path = path
        with open(path, "rb") as f:
            self.b = f.read()
        self.at = 0

    def take(self, n):
        if self.at + n > len(self.b):
            raise RuntimeError(f"{self.path}: truncated file")
        v = self.b[self.at:self.at + n]
        self.at += n
        return v

    def magic(self, m):
        if self.take(4) != m.encode():
            raise RuntimeError(f"{self.path}: bad magic, expected {m}")

    def u32(self):
        return struct.unpack("<I", self.take(4))[0]

    def f64(self):
        return struct.unpack("<d", self.take(8))[0]

    def f64s(self, n):
        return np.frombuffer(self.take(8 * n), dtype="<f8").astype(np.float64)

    def eof(self):
        if self.at != len(self.b):
            raise RuntimeError(f"{self.path}: trailing bytes")


# ---------------------------------------------------------------------------
# SPHF field series (grid.cpp:69-106)
# ---------------------------------------------------------------------------
def write_sphf(path, data, band_limit=0):
    """Write a (t, theta, phi) or (r, t, theta, phi) array as a field series file."""
    a = np.ascontiguousarray(data, dtype=np.float64)
    if a.ndim == 3:
        a = a[None]
    if a.ndim != 4:
        raise ValueError("expected a (t, theta, phi) or (r, t, theta, phi) array")
    if not np.isfinite(a).all():
        raise ValueError("series contains non-finite samples")
    r_len, t_len, nt, nphi = a.shape
    w = _Writer(path)
    w.magic("SPHF")
    for v in (_SPHF_VERSION, nt, nphi, band_limit, t_len, r_len):
        w.u32(v)
    w.f64s(a)
    w.close()


def read_sphf(path):
    """Read a gridded field series; returns (array, band_limit) with the
    array (t, theta, phi) for one replicate, else (r, t, theta, phi)."""
    r = _Reader(path)
    r.magic("SPHF")
    if r.u32() != _SPHF_VERSION:
        raise RuntimeError(f"{path}: unsupported SPHF version")
    nt, nphi, band_limit, t_len, r_len = (r.u32() for _ in range(5))
    if nt < 2 or nphi < 1 or t_len < 1 or r_len < 1:
        raise RuntimeError(f"{path}: implausible SPHF dimensions")
    a = r.f64s(r_len * t_len * nt * nphi).reshape(r_len, t_len, nt, nphi)
    r.eof()
    if band_limit > 0 and band_limit > S.max_band_limit(nt, nphi):
        raise RuntimeError(f"{path}: band limit exceeds what the grid resolves")
    return (a[0] if r_len == 1 else a), band_limit


# ---------------------------------------------------------------------------
# the emulator
# ---------------------------------------------------------------------------
class Emulator:
    """Trained model plus the device state to draw from it (module.cpp:140-179).

    Model parts (stochastic.hpp:71-79): trend records (points x (5 + 2K)),
    lag coefficients phi (order x L^2), the innovation factor as a
    device-resident tiled Cholesky handle (with u_hat and the nugget), and
    the noise variance v2 (points)."""

    def __init__(self, n_theta, n_phi, band_limit, harmonics, period, records, phi, chol, u_hat, nugget,
                 variant, v2, chol_kwargs, diagnostics=None):
        self.n_theta, self.n_phi, self._band_limit = n_theta, n_phi, band_limit
        self.harmonics, self.period = harmonics, period
        self.records, self.phi, self.chol, self.u_hat, self.nugget = records, phi, chol, u_hat, nugget
        self.variant, self.v2, self.chol_kwargs = variant, v2, chol_kwargs
        self.diagnostics = diagnostics or {}
        self._plan = None

    # -- properties of the reference class --------------------------------
    @property
    def band_limit(self):
        return self._band_limit

    @property
    def grid(self):
        return (self.n_theta, self.n_phi)

    def plan(self):
        if self._plan is None:
            self._plan = S.ShtPlan(self.n_theta, self.n_phi, self._band_limit)
        return self._plan

    # -- train (pipeline.cpp:18-54) ----------------------------------------
    @staticmethod
    def train(data, harmonics=2, period=12, var_order=2, band_limit=0, threads=1, variant="dp", tile_size=128,
              band_width_dp=1, sp_fraction=0.05, hp_format="fp16", sp_compute="fp64"):
        """Fit trend, lag and innovation models to a gridded series
        ((t, theta, phi) or (r, t, theta, phi)). threads is accepted for API
        parity; the GPU arguments after it are appended with the reference's
        defaults (TrainConfig: chol dp, tile 128)."""
        import torch
        x = np.ascontiguousarray(data, dtype=np.float64)
        if x.ndim == 3:
            x = x[None]
        if x.ndim != 4:
            raise ValueError("expected a (t, theta, phi) or (r, t, theta, phi) array")
        if not np.isfinite(x).all():
            raise ValueError("series contains non-finite samples")
        r_len, t_len, nt, nphi = x.shape
        L = band_limit if band_limit > 0 else S.max_band_limit(nt, nphi)
        if L > S.max_band_limit(nt, nphi):
            raise ValueError(f"training grid does not resolve band limit {L}")
        points, d = nt * nphi, L * L
        lib = S.lib()
        dev = torch.device("cuda")
        vp = C.c_void_p
        series = torch.from_numpy(x).to(dev)
        # trend (trend.cpp:129-250) and the standardized series
        stride = 5 + 2 * harmonics
        records = np.empty((points, stride))
        S._check(lib.sphemu_gpu_fit_trend(vp(series.data_ptr()), S.DEVICE, r_len, t_len, points, harmonics, period,
                                          S._ptr(records), S.HOST))
        std = torch.empty_like(series)
        S._check(lib.sphemu_gpu_detrend(vp(series.data_ptr()), S.DEVICE, r_len, t_len, S._ptr(records), points,
                                        harmonics, period, None, 0, None, 0, 1, vp(std.data_ptr()), S.DEVICE))
        del series
        # forward SHT of every slice (sht.cpp:374-388)
        plan = S.ShtPlan(nt, nphi, L)
        coeffs = torch.empty((r_len, t_len, d), dtype=torch.float64, device=dev)
        plan.forward_device(std.data_ptr(), r_len * t_len, coeffs.data_ptr())
        # lag model (stochastic.cpp:30-107), residuals left in HBM
        order = var_order
        rows = r_len * (t_len - order) if order > 0 else r_len * t_len
        phi = np.zeros((max(order, 0), d))
        se = np.zeros((max(order, 0), d))
        resid = torch.empty((rows, d), dtype=torch.float64, device=dev)
        zc, uc, nrm = C.c_int64(), C.c_int64(), C.c_double()
        S._check(lib.sphemu_gpu_fit_var(vp(coeffs.data_ptr()), S.DEVICE, r_len, t_len, d, order,
                                        S._ptr(phi) if order > 0 else None, S._ptr(se) if order > 0 else None,
                                        vp(resid.data_ptr()), S.DEVICE, C.byref(zc), C.byref(uc), C.byref(nrm)))
        # innovation covariance + nugget loop, factor kept on the device (stochastic.cpp:109-172)
        kw = dict(variant=variant, tile_size=tile_size, band_width_dp=band_width_dp, sp_fraction=sp_fraction,
                  hp_format=hp_format, sp_compute=sp_compute)
        chol, u_hat, nug = _innovation_factor(resid, r_len, t_len, order, d, kw)
        del resid
        # noise field of what the truncated reconstruction cannot carry (pipeline.cpp:41-42)
        recon = torch.empty_like(std)
        plan.inverse_device(coeffs.data_ptr(), r_len * t_len, recon.data_ptr())
        v2 = np.empty(points)
        S._check(lib.sphemu_gpu_noise_field(vp(std.data_ptr()), vp(recon.data_ptr()), S.DEVICE, r_len * t_len,
                                            points, S._ptr(v2), S.HOST))
        diag = {"zeroed_var_series": zc.value, "unstable_var_series": uc.value, "nugget": nug,
                "residual_mean_norm": nrm.value, "collinear_warnings": 0}
        em = Emulator(nt, nphi, L, harmonics, period, records, phi, chol, u_hat, nug, variant, v2, kw, diag)
        em._plan = plan
        return em

    # -- emulate (stochastic.cpp:217-277) -----------------------------------
    def emulate(self, t_out, seed=1, replicates=1, threads=1, t_start=1, rng="reference", forcing=None):
        """Draw replicate series; returns an (r, t, theta, phi) array. The
        default rng reproduces the reference's serial mt19937_64 stream."""
        plan = self.plan()
        d = self._band_limit ** 2
        phi = self.phi if self.phi.shape[0] else np.zeros((1, d))
        f, fa = S._forcing_args(forcing)
        out = np.empty((replicates, t_out, self.n_theta, self.n_phi))
        S._check(S.lib().sphemu_gpu_emulate_chol_trend(
            self.chol.h, plan.h, S._ptr(phi), self.phi.shape[0], S._ptr(self.records), self.harmonics, self.period,
            *fa, t_start, S._ptr(self.v2), t_out, seed, 0, replicates, {"reference": 0, "philox": 1}[rng],
            S._ptr(out), S.HOST))
        return out

    # -- bundle I/O (pipeline.cpp:56-97) -------------------------------------
    def factor(self):
        """The dense lower factor V of u_hat + nugget I (stored tiles, widened)."""
        return self.chol.factor_dense()

    def save(self, dir):
        d = self._band_limit ** 2
        if d > (1 << 16):
            raise ValueError("UCOV stores at most 65 536 coefficients (band limit 256)")  # stochastic.cpp:327
        os.makedirs(dir, exist_ok=True)
        w = _Writer(os.path.join(dir, "trend.bin"))
        w.magic("TRND")
        for v in (self._band_limit, self.n_theta, self.n_phi, self.harmonics, self.period):
            w.u32(v)
        w.f64s(self.records)
        w.close()
        w = _Writer(os.path.join(dir, "var.bin"))
        w.magic("VARM")
        w.u32(self.phi.shape[0])
        w.u32(self._band_limit)
        w.f64s(self.phi)
        w.close()
        v = self.factor()
        il = np.tril_indices(d)
        w = _Writer(os.path.join(dir, "ucov.bin"))
        w.magic("UCOV")
        w.u32(d)
        w.f64(self.nugget)
        w.f64s(v[il])
        w.u32(_VARIANTS.index(self.variant))
        w.f64s(self.u_hat[il])
        w.close()
        w = _Writer(os.path.join(dir, "noise.bin"))
        w.magic("NOIS")
        w.u32(self.n_theta)
        w.u32(self.n_phi)
        w.f64s(self.v2)
        w.close()
        prov = {"format": "sphemu-bundle-v1", "tool_version": VERSION, "band_limit": self._band_limit,
                "grid": {"n_theta": self.n_theta, "n_phi": self.n_phi},
                "trend": {"harmonics": self.harmonics, "period": self.period}, "var_order": int(self.phi.shape[0]),
                "innovation": {"nugget": self.nugget, "variant": self.variant},
                "chol": {"variant": self.chol_kwargs["variant"], "tile_size": self.chol_kwargs["tile_size"],
                         "band_width_dp": self.chol_kwargs["band_width_dp"],
                         "sp_fraction": self.chol_kwargs["sp_fraction"]}}
        with open(os.path.join(dir, "provenance.json"), "w") as f:
            f.write(json.dumps(prov, indent=2) + "\n")

    @staticmethod
    def load(dir):
        r = _Reader(os.path.join(dir, "trend.bin"))
        r.magic("TRND")
        trend_l, nt, nphi, harmonics, period = (r.u32() for _ in range(5))
        records = r.f64s(nt * nphi * (5 + 2 * harmonics)).reshape(nt * nphi, -1)
        r.eof()
        r = _Reader(os.path.join(dir, "var.bin"))
        r.magic("VARM")
        order, L = r.u32(), r.u32()
        phi = r.f64s(order * L * L).reshape(order, L * L)
        r.eof()
        if trend_l not in (0, L):
            raise RuntimeError(f"{dir}: trend and lag model disagree on the band limit")
        r = _Reader(os.path.join(dir, "ucov.bin"))
        r.magic("UCOV")
        d = r.u32()
        nug = r.f64()
        il = np.tril_indices(d)
        v = np.zeros((d, d))
        v[il] = r.f64s(d * (d + 1) // 2)
        variant = _VARIANTS[r.u32()]
        u = np.zeros((d, d))
        u[il] = r.f64s(d * (d + 1) // 2)
        u = u + np.tril(u, -1).T
        r.eof()
        r = _Reader(os.path.join(dir, "noise.bin"))
        r.magic("NOIS")
        if (r.u32(), r.u32()) != (nt, nphi):
            raise RuntimeError(f"{dir}: noise field has the wrong size")
        v2 = r.f64s(nt * nphi)
        r.eof()
        kw = {"variant": variant, "tile_size": 128, "band_width_dp": 1, "sp_fraction": 0.05}
        p = os.path.join(dir, "provenance.json")
        if os.path.exists(p):
            kw.update(json.load(open(p)).get("chol", {}))
        kw.setdefault("hp_format", "fp16")
        chol = S.Cholesky(d, kw["variant"], tile_size=kw["tile_size"], band_width_dp=kw["band_width_dp"],
                          sp_fraction=kw["sp_fraction"], hp_format=kw["hp_format"])
        S._check(S.lib().sphemu_gpu_chol_load_factor(chol.h, S._ptr(np.ascontiguousarray(v)), S.HOST, d))
        return Emulator(nt, nphi, L, harmonics, period, records, phi, chol, u, nug, variant, v2, kw)


def _innovation_factor(resid, r_len, t_len, order, d, kw):
    cfg = S.make_config(kw["variant"], kw["tile_size"], 1, kw["band_width_dp"], kw["sp_fraction"], kw["hp_format"],
                        "tensor", 1, kw["sp_compute"])
    u = np.empty((d, d))
    nug = C.c_double()
    st = S.CholStats()
    h = C.c_void_p()
    S._check(S.lib().sphemu_gpu_innovation_factor(C.c_void_p(resid.data_ptr()), S.DEVICE, resid.shape[0], d, r_len,
                                                  t_len, order, C.byref(cfg), S._ptr(u), S.HOST, C.byref(nug),
                                                  C.byref(st), C.byref(h)))
    chol = S.Cholesky.__new__(S.Cholesky)
    chol.n, chol.cfg, chol.h, chol.rank, chol.dist = d, cfg, h, 0, None
    return chol, u, nug.value
