mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_trend.py tests/test_gpu_emulate.py -x -q > gpurun_out/pytest_trend5.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_trend5.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:k_trend --log-file gpurun_out/trend_launches5.csv python tools/trend_bench.py > gpurun_out/ncu_trend5.log 2>&1; echo "EXIT $?" >> gpurun_out/ncu_trend5.log
