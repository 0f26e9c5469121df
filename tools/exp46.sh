R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $R tools/dist_timeline.py 129600 512 dpsphp bf16 2 400 2>&1 | grep -v "^W\|NCCL\|Warn\|warn\|return func\|\*\*\*" | head -80
for r in 16 32 64; do echo "reserve $r"; SPHEMU_DIST_RESERVE=$r timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 2 2>&1 | grep "TFLOP"; done
echo "p2p"; SPHEMU_XCHG=p2p timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 2 2>&1 | grep "TFLOP"
echo "4x1"; timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 4 2>&1 | grep "TFLOP"
echo "1x4"; timeout 600 $R tools/dist_perf.py 129600 512 dpsphp bf16 1 2>&1 | grep "TFLOP"
