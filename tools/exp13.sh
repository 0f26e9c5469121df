for y in 0 1; do echo "YIELD=$y"; SPHEMU_YIELD=$y timeout 300 python tools/ab.py 32400 dpsp fp16 5; done
for y in 0 1; do echo "YIELD=$y C3"; SPHEMU_YIELD=$y timeout 300 python tools/ab.py 129600 dpsphp bf16 2; done
for re in 8 16; do for rt in 16 32 48; do echo "early=$re tail=$rt"; SPHEMU_YIELD=0 SPHEMU_RESERVE_EARLY=$re SPHEMU_RESERVE_TAIL=$rt timeout 300 python tools/ab.py 32400 dpsp fp16 3; done; done
timeout 900 python -m pytest tests/test_gpu_chol.py -q -x -p no:cacheprovider -k "lookahead or acceptance or tensor_path" 2>&1 | tail -3
