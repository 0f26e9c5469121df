R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ozaki.py -q -x 2>&1 | tail -2
timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 2 2>&1 | grep "TFLOP"
SPHEMU_DP_EMU=0 timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 2 2>&1 | grep "TFLOP"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534"
timeout 600 $R2 tools/dist_perf.py 129600 512 dpsphp bf16 2 2>&1 | grep "TFLOP"
timeout 300 python tools/ab.py 32400 dpsp fp16 3
timeout 300 python tools/ab.py 129600 dpsphp bf16 2
