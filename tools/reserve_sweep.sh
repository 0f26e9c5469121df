# chain reserve sweep (SPHEMU_RESERVE_EARLY / SPHEMU_RESERVE_TAIL), C2 and C3 on one GPU
python tools/ab.py 32400 dpsp fp16 3
for re in 16 24; do for rt in 8 16 32; do
  echo "early=$re tail=$rt"; SPHEMU_RESERVE_EARLY=$re SPHEMU_RESERVE_TAIL=$rt python tools/ab.py 32400 dpsp fp16 3
done; done
python tools/ab.py 129600 dpsphp bf16 1
for re in 12 16 24; do for rt in 4 16; do
  echo "early=$re tail=$rt"; SPHEMU_RESERVE_EARLY=$re SPHEMU_RESERVE_TAIL=$rt python tools/ab.py 129600 dpsphp bf16 1
done; done
