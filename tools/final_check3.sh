mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_var.py -x -q > gpurun_out/pytest_var4.log 2>&1; echo "PYTEST_EXIT $?" >> gpurun_out/pytest_var4.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_fit_var --log-file gpurun_out/var_launches4.csv python tools/var_bench.py > gpurun_out/ncu_var4.log 2>&1; echo "EXIT $?" >> gpurun_out/ncu_var4.log
timeout 900 python bench.py > gpurun_out/bench_n1_final3.json 2> gpurun_out/bench_n1_final3.err; echo "BENCH_EXIT $?" >> gpurun_out/bench_n1_final3.err
