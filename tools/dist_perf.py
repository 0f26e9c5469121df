"""Distributed Cholesky timing for a given (n, b, variant, hp) over all ranks."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
sph._sphemu.lib().sphemu_gpu_set_device(local)
dist.init_process_group("nccl")
n, b, v, hp = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
P = int(sys.argv[5]) if len(sys.argv) > 5 else world
Q = world // P
obj = [sph.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
h = sph.Cholesky(n, v, tile_size=b, hp_format=hp, dist=(P, Q, rank, obj[0]) if world > 1 else None)
fl = h.flops()
for rep in range(2):
    h.generate_spd(1)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.factor()
    st = h.wait()
    dist.barrier()
    dt = time.perf_counter() - t0
probe = h.residual_probe(1, 2)
if rank == 0:
    print(f"n={n} b={b} {v}/{hp} {P}x{Q}: {dt*1e3:.1f} ms  {n**3/3/dt/1e12:.1f} TFLOP/s total  probe {probe:.2e} "
          f"flops {({k: round(x/1e12, 2) for k, x in fl.items()})}", flush=True)
dist.destroy_process_group()
