SPHEMU_LAUNCH_LOG=1 timeout 300 python tools/chol_once.py 32400 512 dpsp 1 2> gpurun_out/launch_log_c2.txt > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:"k_tc_gemm<256, 3, 0, 2>" -s 20 -o gpurun_out/ncu_sp_pair -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:k_oz_update -s 30 -o gpurun_out/ncu_oz_c2 -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2_r02c.csv python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:"k_tc_gemm<256, 1, 0, 2>" -s 200 -o gpurun_out/ncu_hp_pair -f python tools/chol_once.py 64800 512 dpsphp 1 > /dev/null 2>&1
ls -la gpurun_out | tail -6
