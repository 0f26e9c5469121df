python -m pytest tests/test_gpu_chol.py -q -x 2>&1 | tail -2
SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16
python tools/epi_probe.py 98304 dpsphp bf16
python tools/epi_probe.py 32400 dpsp fp16
