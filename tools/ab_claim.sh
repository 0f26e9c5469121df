for lib in paper_2408_04440_b200/lib/libsphemu_gpu.so variants/claim/libsphemu_gpu.so; do
  SPHEMU_LIB=$lib python tools/ab.py 32400 dpsp fp16 4
  SPHEMU_LIB=$lib python tools/ab.py 129600 dpsphp bf16 2
done
SPHEMU_TC_CG=2 python tools/ab.py 129600 dpsphp bf16 2
