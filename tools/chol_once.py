"""One warm factorization of make_spd_test_matrix(n, 1) (for ncu launch lists):
tools/chol_once.py N B VARIANT [REPS] [HP_FORMAT]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

n, b, v = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
hp = sys.argv[5] if len(sys.argv) > 5 else "fp16"
h = sph.Cholesky(n, v, tile_size=b, hp_format=hp)
for _ in range(int(sys.argv[4]) if len(sys.argv) > 4 else 2):
    h.generate_spd(1)
    h.factor()
    st = h.wait()
print(f"n={n} b={b} {v} {st.device_ms:.2f} ms {n**3/3/st.device_ms/1e9:.1f} TFLOP/s")
