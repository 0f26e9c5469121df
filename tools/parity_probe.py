"""Parity probe where the flops are: dense, non-decaying SPD inputs and the
C1-style nugget-regularised covariance through the b=256/512 tensor path.
Prints one JSON line per case: GPU residual, oracle residual, ratio and the
elementwise distance to the oracle factor (scaled by max|L|)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
import paper_2408_04440_b200 as sph  # noqa: E402


def dense_spd(d, seed, ratio=2.0, delta=1e-3):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((int(ratio * d), d))
    a = x.T @ x / x.shape[0]
    a = 0.5 * (a + a.T)
    a[np.diag_indices(d)] += delta
    return a


def kms_spd(d, seed, rho):
    """make_spd_test_matrix with the 0.9 decay replaced by rho (rho -> 1: O(1) tiles everywhere)."""
    a = O.make_spd(d, seed)
    dd = np.sqrt(np.diag(a) / 1.25)
    i = np.arange(d)
    a = 0.25 * np.outer(dd, dd) * rho ** np.abs(i[:, None] - i[None, :])
    a[i, i] = 1.25 * dd * dd
    return a


def case(name, a, variant, b, **kw):
    t0 = time.time()
    f, _ = sph.tiled_cholesky(a, variant, tile_size=b, **kw)
    okw = {k: v for k, v in kw.items() if k in ("hp_format", "band_width_dp", "sp_fraction")}
    ref, _ = O.tiled_cholesky(a, variant, tile_size=b, workers=os.cpu_count() or 8, **okw)
    rg, ro = O.relative_residual(a, f), O.relative_residual(a, ref)
    scale = np.abs(ref).max()
    out = dict(case=name, variant=variant, b=b, n=a.shape[0], **kw, r_gpu=rg, r_ref=ro, ratio=rg / ro,
               elem=float(np.abs(f - ref).max() / scale), s=round(time.time() - t0, 1))
    print(json.dumps(out), flush=True)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "dense"):
        for d, b in ((2048, 256), (3072, 512)):
            a = dense_spd(d, 11)
            for v in ("dp", "dpsp", "dpsphp", "dphp"):
                for hp in ("fp16", "bf16") if v in ("dpsphp", "dphp") else ("fp16",):
                    for spc in ("fp16x3", "tf32x3") if v in ("dpsp", "dpsphp") else ("fp16x3",):
                        case("dense_xtx", a, v, b, hp_format=hp, sp_compute=spc)
    if which in ("all", "kms"):
        for rho in (0.999, 0.9999):
            a = kms_spd(3072, 1, rho)
            for v in ("dpsp", "dpsphp", "dphp"):
                for hp in ("fp16", "bf16") if v != "dpsp" else ("fp16",):
                    case(f"kms_{rho}", a, v, 512, hp_format=hp)
    if which in ("all", "nugget"):
        import ctypes as C
        rng = np.random.default_rng(91)
        d = 2025
        n = 97
        for rank in (97, 40):
            basis = rng.standard_normal((rank, d)) / (1.0 + np.arange(d) % 45) ** 0.5
            xi = rng.standard_normal((n, rank)) @ basis
            for v in ("dp", "dpsp", "dpsphp", "dphp"):
                for b in (256, 512):
                    u, vv, nug, _ = sph._sphemu.estimate_innovation_covariance(xi, 1, n + 3, 3, variant=v,
                                                                               tile_size=b)
                    uo = np.empty((d, d))
                    vo = np.empty((d, d))
                    nugo = C.c_double()
                    st = O.CholStats()
                    cfg = O.config(v, b)
                    rc = O.lib().so_estimate_innovation_covariance(np.ascontiguousarray(xi), n, d, C.byref(cfg),
                                                                   1, uo, vo, C.byref(nugo), C.byref(st))
                    tgt = u + nug * np.eye(d)
                    rg = O.relative_residual(tgt, vv)
                    tgo = uo + nugo.value * np.eye(d)
                    ro = O.relative_residual(tgo, vo)
                    print(json.dumps(dict(case=f"nugget_rank{rank}", variant=v, b=b, nug=nug, nug_ref=nugo.value,
                                          rc=rc, r_gpu=rg, r_ref=ro, ratio=rg / ro)), flush=True)


if __name__ == "__main__":
    main()
