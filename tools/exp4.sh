timeout 900 python -m pytest tests/test_gpu_emulate_chol.py -q -x -p no:cacheprovider > gpurun_out/pytest_emul_chol.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_emul_chol.log
tail -5 gpurun_out/pytest_emul_chol.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_parity.log
tail -8 gpurun_out/pytest_parity.log
