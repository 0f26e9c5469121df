mkdir -p gpurun_out
timeout 300 python tools/var_bench.py > gpurun_out/var_bench.log 2>&1; echo "EXIT $?" >> gpurun_out/var_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_bytes.sum --clock-control none --csv -k regex:k_fit_var --log-file gpurun_out/var_launches.csv python tools/var_bench.py > gpurun_out/ncu_var.log 2>&1; echo "EXIT $?" >> gpurun_out/ncu_var.log
