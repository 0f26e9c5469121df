"""Re-time single parts of the bench line in isolation (development aid):
tools/bench_parts.py c1|emul [L]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2408_04440_b200 as sph  # noqa: E402

what = sys.argv[1]
if what == "c1":
    for _ in range(2):
        r = bench.c1_point(sph)
        print("c1 gpu_s", {k: round(v, 3) for k, v in r["gpu_s"].items()}, "cpu total", round(r["cpu_s"]["total"], 2))
else:
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 180
    h = sph.Cholesky(L * L, "dpsp", tile_size=512)
    h.generate_spd(1)
    h.factor()
    h.wait()
    for _ in range(3):
        t0 = time.perf_counter()
        r = bench.emulation_point(sph, h, L)
        print("emul", L, round(r["snapshots_per_s"]), round(r["seconds"], 4), "wall", round(time.perf_counter() - t0, 2))
