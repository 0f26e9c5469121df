mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_trend.py tests/test_gpu_emulate.py -x -q > gpurun_out/pytest_trend2.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_trend2.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_trend --log-file gpurun_out/trend_launches2.csv python tools/trend_bench.py > gpurun_out/ncu_trend3.log 2>&1; echo "EXIT $?" >> gpurun_out/ncu_trend3.log
