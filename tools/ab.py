"""A/B helper: factor make_spd_test_matrix(n, 1) a few times with the library
SPHEMU_LIB points at; print the best device time, TFLOP/s and the residual
probe (tools/ab.py N VARIANT HP_FORMAT [REPS] [TILE])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, v, hp = int(sys.argv[1]), sys.argv[2], sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
tile = int(sys.argv[5]) if len(sys.argv) > 5 else 512
h = sph.Cholesky(n, v, tile_size=tile, hp_format=hp)
ts = []
for _ in range(reps + 1):
    h.generate_spd(1)
    h.factor()
    ts.append(h.wait().device_ms)
best = min(ts[1:])
print(f"{os.environ.get('SPHEMU_LIB', 'default')}: n={n} b={tile} {v}/{hp} best {best:.2f} ms "
      f"({n**3/3/best/1e9:.1f} TFLOP/s) all={[round(t, 1) for t in ts[1:]]} probe={h.residual_probe(1, 2):.2e}")
