timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1 -k regex:"k_tc_gemm<256, 3, 0, 2>" -s 20 -o gpurun_out/ncu_sp_pair -f python tools/chol_once.py 32400 512 dpsp 1 > gpurun_out/ncu_sp_pair.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -c 1 -k regex:"k_tc_gemm<256, 1, 0, 2>" -s 200 -o gpurun_out/ncu_hp_pair -f python tools/chol_once.py 64800 512 dpsphp 1 > gpurun_out/ncu_hp_pair.log 2>&1
SPHEMU_LAUNCH_LOG=1 timeout 300 python tools/chol_once.py 64800 512 dpsphp 1 2> gpurun_out/launch_log_64800.txt > /dev/null
tail -3 gpurun_out/ncu_sp_pair.log
