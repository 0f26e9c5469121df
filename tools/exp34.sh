echo "epi4"; timeout 60 ./tools/micro/oz_bench; echo "epi8"; LD_LIBRARY_PATH=$PWD/build_alt timeout 60 ./tools/micro/oz_bench
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x 2>&1 | tail -2
timeout 300 python tools/ab.py 32400 dpsp fp16 4
timeout 300 python tools/ab.py 129600 dpsphp bf16 2
timeout 300 python tools/ab.py 64800 dpsp fp16 2
timeout 300 python tools/chol_timeline.py 32400 512 dpsp 2>/dev/null | head -9
