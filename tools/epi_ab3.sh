# register-staged C vs the TMA ring (variants: regc_epi8 = -DSPH_TC_EPI16=0, tma = -DSPH_TC_REGC=0)
python -m pytest tests/test_gpu_chol.py -q -x 2>&1 | tail -2
SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16
SPHEMU_LIB=variants/regc_epi8/libsphemu_gpu.so SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16
SPHEMU_LIB=variants/tma/libsphemu_gpu.so SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16
SPHEMU_TC_CG=1 python tools/epi_probe.py 98304 dpsphp bf16
python tools/epi_probe.py 32400 dpsp fp16
SPHEMU_LIB=variants/tma/libsphemu_gpu.so python tools/epi_probe.py 32400 dpsp fp16
python tools/ab.py 32400 dpsp fp16 3
SPHEMU_TC_CG=2 python tools/ab.py 129600 dpsphp bf16 2
