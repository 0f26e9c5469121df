export SPHEMU_YIELD=0
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1 -k 'regex:k_tc_gemm<\(int\)256, \(int\)3, \(int\)0, \(int\)2>' -s 44 -o gpurun_out/ncu_sp_pair_v2 -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
SPHEMU_TC_OPT=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 1 -k 'regex:k_tc_gemm<\(int\)256, \(int\)3, \(int\)0, \(int\)2>' -s 44 --csv --log-file gpurun_out/sp_pair_prefetch_on.csv python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
unset SPHEMU_YIELD
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1 -k 'regex:k_tc_gemm<\(int\)256, \(int\)1, \(int\)0, \(int\)2>' -s 300 -o gpurun_out/ncu_hp_pair_c3 -f python tools/chol_once.py 129600 512 dpsphp 1 bf16 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2_r02d.csv python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
