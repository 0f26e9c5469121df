timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:k_oz_update -s 20 -o gpurun_out/ncu_oz_dp -f python tools/chol_once.py 16384 512 dp 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2_oz.csv python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
ls -la gpurun_out/ | tail -3
