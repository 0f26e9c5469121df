timeout 900 python -m pytest tests/test_gpu_emulate_chol.py tests/test_gpu_emulate.py -q -p no:cacheprovider 2>&1 | tail -8
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_try.json 2> gpurun_out/bench_try.err; echo "BENCH EXIT $?"
tail -5 gpurun_out/bench_try.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_try.json 2> gpurun_out/bench_ref_try.err; echo "REF EXIT $?"
