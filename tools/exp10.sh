# ncu captures: one launch each of the kernels the verdict asks for (C2 factor, C4 SHT, L=180 emulation)
set -x
N="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $N -k regex:k_potrf_coop -s 20 -o gpurun_out/ncu_potrf -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_update_fp64_v2 -s 20 -o gpurun_out/ncu_dpupd -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_tc_gemm -s 30 -o gpurun_out/ncu_spupd -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_panel_prep -s 10 -o gpurun_out/ncu_panelprep -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_load_dense -s 0 -o gpurun_out/ncu_load -f python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_ring_rfft_fwd -s 1 -o gpurun_out/ncu_rfft_fwd -f python tools/sht_once.py 721 1440 720 1000 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_ring_rfft_inv -s 1 -o gpurun_out/ncu_rfft_inv -f python tools/sht_once.py 721 1440 720 1000 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_legendre_fwd -s 1 -o gpurun_out/ncu_leg_fwd -f python tools/sht_once.py 721 1440 720 1000 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_legendre_inv -s 1 -o gpurun_out/ncu_leg_inv -f python tools/sht_once.py 721 1440 720 1000 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_legendre_fwd -s 1 -o gpurun_out/ncu_leg_fwd_c2 -f python tools/sht_once.py 181 360 180 1000 1 > /dev/null 2>&1
timeout 600 $N -k regex:k_tc_trmm -s 1 -o gpurun_out/ncu_trmm -f python tools/emul_once.py 180 dpsphp > /dev/null 2>&1
timeout 600 $N -k regex:k_trmm_dp -s 1 -o gpurun_out/ncu_trmm_dp -f python tools/emul_once.py 180 dpsphp > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/chol_once.py 32400 512 dpsp 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_emul.csv python tools/emul_once.py 180 dpsphp > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests/test_cpp_api.py -q -p no:cacheprovider 2>&1 | tail -3
