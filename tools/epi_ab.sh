# A/B of the update epilogue layouts (tools/build_variant.sh epi8 -DSPH_TC_EPI16=0, epi16r2 -DSPH_TC_RING16=2)
for cg in 1 2; do
  SPHEMU_LIB=variants/epi8/libsphemu_gpu.so SPHEMU_TC_CG=$cg python tools/epi_probe.py 98304 dpsphp bf16
  SPHEMU_TC_CG=$cg python tools/epi_probe.py 98304 dpsphp bf16
done
SPHEMU_LIB=variants/epi16r2/libsphemu_gpu.so SPHEMU_TC_CG=2 python tools/epi_probe.py 98304 dpsphp bf16
for cg in 1 2; do SPHEMU_TC_CG=$cg python tools/ab.py 129600 dpsphp bf16 2; done
python -m pytest tests/test_gpu_chol.py -q -x 2>&1 | tail -2
