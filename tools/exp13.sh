for y in 0 1; do echo "YIELD=$y"; SPHEMU_YIELD=$y timeout 300 python tools/ab.py 32400 dpsp fp16 5; done
for y in 0 1; do echo "YIELD=$y C3"; SPHEMU_YIELD=$y timeout 300 python tools/ab.py 129600 dpsphp bf16 2; done
timeout 900 python -m pytest tests/test_gpu_chol.py tests/test_gpu_sht.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python - <<'PY'
import sys, time, json
sys.path.insert(0, '.')
import bench, paper_2408_04440_b200 as sph
print(json.dumps(bench.sht_c4(sph, 1000, 8760))[:1500])
PY
./tools/micro/potrf_trace 2>&1 | tail -45
