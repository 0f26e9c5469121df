"""Per-step timeline of the lookahead schedule (chain vs bulk stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, b, v = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
hp = sys.argv[4] if len(sys.argv) > 4 else "fp16"
h = sph.Cholesky(n, v, tile_size=b, hp_format=hp)
h.set_profiling(True)
for _ in range(2):
    h.generate_spd(1)
    h.factor()
    st = h.wait()
tl = h.timeline()
print(f"total {st.device_ms:.2f} ms")
busy = {0: 0.0, 1: 0.0}
for ph, s, a, z in tl:
    busy[s] += z - a
print("stream busy ms: bulk %.1f chain %.1f" % (busy[0], busy[1]))
# chain gaps: for each step the chain span = from its first op to its last op
import collections
agg = collections.defaultdict(float)
for ph, s, a, z in tl:
    agg[(s, ph)] += z - a
for k, v in sorted(agg.items()):
    print(("bulk " if k[0] == 0 else "chain"), k[1], f"{v:.2f} ms")
# print every 8th step window
last = 0
rows = sorted(tl, key=lambda x: x[2])
for i, (ph, s, a, z) in enumerate(rows):
    if i < 40 or i > len(rows) - 40:
        print(f"{'B' if s == 0 else 'C'} {ph:10s} {a:8.3f} {z:8.3f} {z - a:7.3f}")
