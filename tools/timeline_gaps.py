"""Idle time of the bulk (0) and chain (1) streams per quarter of a profiled
factorization: which stream is the critical one when
(tools/timeline_gaps.py N VARIANT [HP_FORMAT])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, v = int(sys.argv[1]), sys.argv[2]
hp = sys.argv[3] if len(sys.argv) > 3 else "fp16"
h = sph.Cholesky(n, v, tile_size=512, hp_format=hp)
h.set_profiling(True)
for _ in range(2):
    h.generate_spd(1)
    h.factor()
    st = h.wait()
tl = h.timeline()
t_end = max(z for _, _, _, z in tl)
print(f"n={n} {v}: {st.device_ms:.2f} ms, timeline span {t_end:.2f} ms")
for s in (0, 1):
    iv = sorted((a, z) for _, st_, a, z in tl if st_ == s)
    # merge overlapping intervals, then idle per quarter
    merged = []
    for a, z in iv:
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], z)
        else:
            merged.append([a, z])
    q = [0.0] * 4
    for w in range(4):
        lo, hi = t_end * w / 4, t_end * (w + 1) / 4
        busy = sum(max(0.0, min(z, hi) - max(a, lo)) for a, z in merged)
        q[w] = (hi - lo) - busy
    print(("bulk " if s == 0 else "chain") + " idle ms per quarter: " + " ".join(f"{x:6.2f}" for x in q))
