for d in 0 1 2; do echo dbg$d; SPHEMU_OZ_DBG=$d timeout 60 ./tools/micro/oz_bench; done
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x 2>&1 | tail -2
timeout 300 python tools/ab.py 32400 dpsp fp16 4
timeout 300 python tools/ab.py 129600 dpsphp bf16 2
