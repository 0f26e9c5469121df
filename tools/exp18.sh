timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1_r02.json 2> gpurun_out/bench_n1_r02.err; echo "BENCH EXIT $?"; tail -2 gpurun_out/bench_n1_r02.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2_r02.csv python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:k_tc_gemm -s 40 -o gpurun_out/ncu_spupd_merged -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 1 -k regex:"k_tc_gemm<256, 1, 0, 2>" -s 60 -o gpurun_out/ncu_hpupd_merged -f python tools/chol_once.py 64800 512 dpsphp 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | tail -3
