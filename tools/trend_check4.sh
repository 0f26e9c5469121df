mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_trend.py tests/test_gpu_emulate.py tests/test_cpp_api.py -x -q > gpurun_out/pytest_trend6.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_trend6.log
timeout 300 python tools/trend_bench.py > gpurun_out/trend_bench6.log 2>&1; echo "EXIT $?" >> gpurun_out/trend_bench6.log
