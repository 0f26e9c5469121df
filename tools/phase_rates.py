"""Per-class update rates of one factorization (profiled phases): the update
kernels' achieved TFLOP/s at a given tile size (is the C round trip binding?).
tools/phase_rates.py N VARIANT HP B"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, v, hp, b = int(sys.argv[1]), sys.argv[2], sys.argv[3], int(sys.argv[4])
h = sph.Cholesky(n, v, tile_size=b, hp_format=hp)
h.generate_spd(1)
h.factor()
st = h.wait()
h.set_profiling(True)
h.reset_phase_times()
h.generate_spd(1)
h.factor()
st = h.wait()
ph = h.phase_times()
f = h.class_update_flops()
out = {"n": n, "b": b, "variant": v, "hp": hp, "device_ms": st.device_ms}
for c in ("dp", "sp", "hp"):
    ms = ph["update_" + c]["ms"]
    if ms > 0:
        out["update_" + c] = {"ms": ms, "tflops": f[c] / (ms * 1e-3) / 1e12}
out["potrf_ms"] = ph["potrf"]["ms"]
out["panel_ms"] = ph["panel"]["ms"]
print(json.dumps(out), flush=True)
