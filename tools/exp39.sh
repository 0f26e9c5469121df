export SPHEMU_YIELD=0
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1 -k 'regex:k_tc_gemm<\(int\)256, \(int\)3, \(int\)0, \(int\)2>' -s 44 -o gpurun_out/ncu_sp_pair -f python tools/chol_once.py 32400 512 dpsp 1 > gpurun_out/ncu_sp_pair.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:k_oz_update -s 44 -o gpurun_out/ncu_oz_c2 -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1 -k 'regex:k_tc_gemm<\(int\)256, \(int\)1, \(int\)0, \(int\)2>' -s 104 -o gpurun_out/ncu_hp_pair -f python tools/chol_once.py 64800 512 dpsphp 1 > gpurun_out/ncu_hp_pair.log 2>&1
SPHEMU_LAUNCH_LOG=1 timeout 300 python tools/chol_once.py 32400 512 dpsp 1 2> gpurun_out/launch_log_c2_noyield.txt > /dev/null
ls gpurun_out/*.ncu-rep
