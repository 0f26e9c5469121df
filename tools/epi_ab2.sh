# pair epilogue layouts at the HP class, then the SP pair at C2
for v in pair8r1 pair8r2; do SPHEMU_LIB=variants/$v/libsphemu_gpu.so SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16; done
SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16
python tools/epi_probe.py 32400 dpsp fp16
SPHEMU_TC_CG_SP=2 python tools/epi_probe.py 32400 dpsp fp16
python tools/ab.py 32400 dpsp fp16 3
SPHEMU_TC_CG_SP=2 python tools/ab.py 32400 dpsp fp16 3
