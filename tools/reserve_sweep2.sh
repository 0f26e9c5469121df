for re in 8 12; do for rt in 32 48; do
  echo "C2 early=$re tail=$rt"; SPHEMU_RESERVE_EARLY=$re SPHEMU_RESERVE_TAIL=$rt python tools/ab.py 32400 dpsp fp16 3
done; done
for re in 8 12; do for rt in 32; do
  echo "C3 early=$re tail=$rt"; SPHEMU_RESERVE_EARLY=$re SPHEMU_RESERVE_TAIL=$rt python tools/ab.py 129600 dpsphp bf16 1
done; done
