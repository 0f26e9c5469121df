run() { port=$((29600 + RANDOM % 1000)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $port tools/dist_perf.py 129600 512 dpsphp bf16 $2 2>&1 | grep "TFLOP" ; }
echo "p2p plain"; run 4 2
echo "bcast plain"; SPHEMU_XCHG=bcast run 4 2
echo "bcast shift"; SPHEMU_XCHG=bcast SPHEMU_MAP=shift run 4 2
echo "p2p shift"; SPHEMU_MAP=shift run 4 2
echo "2gpu p2p"; run 2 2
echo "2gpu bcast"; SPHEMU_XCHG=bcast run 2 2
for r in 16 48; do echo "bcast plain reserve=$r"; SPHEMU_XCHG=bcast SPHEMU_DIST_RESERVE=$r run 4 2; done
