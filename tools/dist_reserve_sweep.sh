# distributed chain-reserve sweep on C3 (2x2 and 2x1 grids)
port=29600
run() { port=$((port+1)); python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $port tools/dist_perf.py 129600 512 dpsphp bf16 $3 2>&1 | grep -v Warn | tail -1; }
echo "4 GPUs default"; run 4 29000 2
for e in 16 24 32; do echo "4 GPUs early=$e"; SPHEMU_DIST_RESERVE_EARLY=$e run 4 0 2; done
echo "2 GPUs default"; CUDA_VISIBLE_DEVICES=0,1 run 2 0 2
for e in 8 16; do echo "2 GPUs early=$e"; CUDA_VISIBLE_DEVICES=0,1 SPHEMU_DIST_RESERVE_EARLY=$e run 2 0 2; done
