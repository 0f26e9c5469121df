timeout 1200 python -m pytest tests/test_gpu_dist.py -q -s -p no:cacheprovider 2>&1 | tail -25
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "BENCH4 EXIT $?"
tail -3 gpurun_out/bench_n4.err
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 tools/c5_run.py 360000 1024 > gpurun_out/c5_n4.json 2> gpurun_out/c5_n4.err; echo "C5 EXIT $?"
tail -3 gpurun_out/c5_n4.err; cat gpurun_out/c5_n4.json
