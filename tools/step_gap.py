"""Where a bench step's time goes beyond the factorization: K back-to-back
(device load + factor) steps timed with CUDA events, with and without the
bench's per-launch profiling, against the load alone and the handle's own
device_ms (tools/step_gap.py [N] [VARIANT] [HP] [K])."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32400
v = sys.argv[2] if len(sys.argv) > 2 else "dpsp"
hp = sys.argv[3] if len(sys.argv) > 3 else "fp16"
K = int(sys.argv[4]) if len(sys.argv) > 4 else 10
g = sph.Cholesky(n, "dp", tile_size=512)
g.generate_spd(1)
a = torch.empty((n, n), dtype=torch.float64, device="cuda")
g.store(a.data_ptr())
del g
a += torch.tril(a, -1).T
torch.cuda.synchronize()
h = sph.Cholesky(n, v, tile_size=512, hp_format=hp)
DEV = sph._sphemu.DEVICE


def run(load=True, factor=True, prof=None):
    if prof is not None:
        h.set_profiling(True, phases=prof)
    else:
        h.set_profiling(False)
    for w in range(3):
        if load:
            h.load(a.data_ptr(), where=DEV, lda=n)
        if factor:
            h.factor()
            h.wait()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dms = []
    e0.record()
    for i in range(K):
        if load:
            h.load(a.data_ptr(), where=DEV, lda=n)
        if factor:
            h.factor()
            st = h.wait() if i == K - 1 else None
    e1.record()
    torch.cuda.synchronize()
    if factor:
        dms.append(st.device_ms)
    return e0.elapsed_time(e1) / K, dms


print("load+factor, no profiling: %.2f ms/step, device_ms %s" % run())
print("load+factor, update_sp events: %.2f ms/step, device_ms %s" % run(prof=["update_" + ("sp" if v == "dpsp" else "hp")]))
h.phase_times(reset=True)
run(prof=["load"])
pt = h.phase_times()["load"]
print("load: %.2f ms per call" % (pt["ms"] / max(1, pt["launches"])))
