mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_var.py tests/test_gpu_trend.py -x -q > gpurun_out/pytest_var.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_var.log
