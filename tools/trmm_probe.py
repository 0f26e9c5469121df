"""Relative error of the tiled innovation product xi = eta L^T against FP64,
per precision class and TMEM flush length (SPHEMU_TRMM_FLUSH_K is read once
per process: run one process per value), plus its speed."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_04440_b200 as sph  # noqa: E402


def dense_spd(d, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((2 * d, d))
    a = x.T @ x / (2 * d)
    a[np.diag_indices(d)] += 1e-3
    return 0.5 * (a + a.T)


n, b, S = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = dense_spd(n, 7)
eta = np.random.default_rng(1).standard_normal((S, n))
for variant, hp in (("dpsp", "fp16"), ("dphp", "fp16"), ("dphp", "bf16")):
    h = sph.Cholesky(n, variant, tile_size=b, hp_format=hp)
    h.load(a)
    h.factor()
    h.wait()
    L = h.factor_dense()
    want = eta @ L.T
    got = h.trmm(eta)
    t0 = time.perf_counter()
    got = h.trmm(eta)
    dt = time.perf_counter() - t0
    err = np.abs(got - want)
    print(json.dumps({"flush_k": os.environ.get("SPHEMU_TRMM_FLUSH_K", "2048"), "variant": variant, "hp": hp,
                      "n": n, "b": b, "S": S, "max_rel": float(err.max() / np.abs(want).max()),
                      "rms_rel": float(np.sqrt((err ** 2).mean() / (want ** 2).mean())), "call_s": dt}), flush=True)
