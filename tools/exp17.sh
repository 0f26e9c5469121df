for m in 1 0; do echo "MERGE=$m"; SPHEMU_MERGE=$m timeout 300 python tools/ab.py 32400 dpsp fp16 4; SPHEMU_MERGE=$m timeout 300 python tools/ab.py 129600 dpsphp bf16 2; done
timeout 300 python tools/phase_rates.py 64800 dpsphp bf16 512
timeout 1200 python -m pytest tests/test_gpu_chol.py tests/test_gpu_parity.py tests/test_gpu_emulate_chol.py tests/test_gpu_covariance.py -q -x -p no:cacheprovider 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -s -p no:cacheprovider 2>&1 | tail -12
