timeout 1200 python -m pytest tests/test_gpu_dist.py -q -s -p no:cacheprovider 2>&1 | tail -15
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "BENCH2 EXIT $?"
tail -3 gpurun_out/bench_n2.err
