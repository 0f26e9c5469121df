for d in 0 1 2; do
SPHEMU_OZ_DBG=$d timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_oz_update -c 6 --csv --log-file gpurun_out/oz_dbg$d.csv python tools/chol_once.py 16384 512 dp 1 > /dev/null 2>&1
done
