timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -3
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 2 2>&1 | grep -v "^W\|NCCL" | tail -4
SPHEMU_DP_EMU=0 timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 2 2>&1 | grep -v "^W\|NCCL" | tail -4
timeout 1500 $R bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_n4_r02b.json 2> gpurun_out/bench_n4_r02b.err; echo "BENCH4 EXIT $?"
