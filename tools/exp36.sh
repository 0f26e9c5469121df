timeout 300 python tools/ab.py 32400 dpsp fp16 4
timeout 300 python tools/ab.py 129600 dpsphp bf16 2
timeout 300 python tools/ab.py 64800 dpsp fp16 2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1_r02b.json 2> gpurun_out/bench_n1_r02b.err; echo "BENCH EXIT $?"
