timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_parity.log
tail -5 gpurun_out/pytest_parity.log
timeout 600 python tools/parity_probe.py nugget > gpurun_out/probe_nugget_a.log 2>&1; echo "EXIT $?" >> gpurun_out/probe_nugget_a.log
SPHEMU_SYNC_CHECK=1 timeout 600 python tools/parity_probe.py nugget > gpurun_out/probe_nugget_b.log 2>&1; echo "EXIT $?" >> gpurun_out/probe_nugget_b.log
tail -3 gpurun_out/probe_nugget_a.log gpurun_out/probe_nugget_b.log
