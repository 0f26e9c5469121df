mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_var.py tests/test_cpp_api.py -x -q > gpurun_out/pytest_var3.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_var3.log
timeout 300 python tools/var_bench.py > gpurun_out/var_bench3.log 2>&1; echo "EXIT $?" >> gpurun_out/var_bench3.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_fit_var --log-file gpurun_out/var_launches3.csv python tools/var_bench.py > gpurun_out/ncu_var3.log 2>&1; echo "EXIT $?" >> gpurun_out/ncu_var3.log
