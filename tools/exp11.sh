for o in 0 4 8 12; do echo "OPT=$o"; SPHEMU_TC_OPT=$o timeout 300 python tools/ab.py 32400 dpsp fp16 5; done
for o in 0 12; do echo "OPT=$o C3"; SPHEMU_TC_OPT=$o timeout 300 python tools/ab.py 129600 dpsphp bf16 2; done
timeout 300 python tools/trmm_probe.py 4096 512 512
timeout 600 ncu --set full --clock-control none -c 1 -k regex:k_tc_gemm -s 30 -o gpurun_out/ncu_spupd2 -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -c 1 -k regex:k_tc_trmm -s 1 -o gpurun_out/ncu_trmm2 -f python tools/emul_once.py 180 dpsphp > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_emulate_chol.py tests/test_cpp_api.py -q -p no:cacheprovider 2>&1 | tail -3
