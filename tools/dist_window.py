"""All ranks' chain / bulk spans of the distributed factorization merged on one
time axis for a window (torchrun; tools/dist_window.py N B VARIANT HP P T0_MS T1_MS)."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
sph._sphemu.lib().sphemu_gpu_set_device(local)
dist.init_process_group("nccl")
n, b, v, hp, P = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
t0, t1 = float(sys.argv[6]), float(sys.argv[7])
obj = [sph.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
h = sph.Cholesky(n, v, tile_size=b, hp_format=hp, dist=(P, world // P, rank, obj[0]))
h.set_profiling(True)
for _ in range(2):
    h.generate_spd(1)
    dist.barrier()
    torch.cuda.synchronize()
    h.factor()
    st = h.wait()
tl = [(rank, ph, s, a, z) for ph, s, a, z in h.timeline() if z >= t0 and a <= t1]
allt = [None] * world
dist.all_gather_object(allt, tl)
if rank == 0:
    rows = sorted((x for part in allt for x in part), key=lambda x: x[3])
    for r, ph, s, a, z in rows:
        if s == 0 and ph.startswith("update") and z - a < 0.02:
            continue
        print(f"r{r} {'BCX'[s]} {ph:10s} {a:9.3f} {z:9.3f} {z - a:7.3f}")
dist.destroy_process_group()
