mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_trend.py tests/test_cpp_api.py -x -q > gpurun_out/pytest_trend.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_trend.log
timeout 300 python tools/trend_bench.py > gpurun_out/trend_bench.log 2>&1; echo "EXIT $?" >> gpurun_out/trend_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_trend --log-file gpurun_out/trend_launches.csv python tools/trend_bench.py > gpurun_out/ncu_trend1.log 2>&1; echo "EXIT $?" >> gpurun_out/ncu_trend1.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_trend -c 1 -o gpurun_out/trend_full python tools/trend_bench.py > gpurun_out/ncu_trend2.log 2>&1; echo "EXIT $?" >> gpurun_out/ncu_trend2.log
