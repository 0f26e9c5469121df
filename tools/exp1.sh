set -x
python tools/parity_probe.py kms > gpurun_out/exp_default.log 2>&1
SPHEMU_PANEL_FP64=1 python tools/parity_probe.py kms > gpurun_out/exp_panel64.log 2>&1
SPHEMU_PANEL_FP64=1 SPHEMU_SP_FP64=1 python tools/parity_probe.py kms > gpurun_out/exp_panel64_sp64.log 2>&1
SPHEMU_SP_FP64=1 python tools/parity_probe.py kms > gpurun_out/exp_sp64.log 2>&1
SPHEMU_PANEL_FP64=1 python tools/parity_probe.py dense > gpurun_out/exp_dense_panel64.log 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/parity_probe.py nugget > gpurun_out/exp_nugget_memcheck.log 2>&1
echo done
