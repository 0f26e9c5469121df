for y in 1 0; do echo "YIELD=$y"; SPHEMU_YIELD=$y timeout 300 python tools/ab.py 32400 dpsp fp16 5; done
SPHEMU_YIELD=1 timeout 300 python tools/chol_timeline.py 32400 512 dpsp 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_chol.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
