"""C5-shaped run (BASELINE configs[4]) on the GPUs of one box (torchrun, one
process per GPU): make_spd_test_matrix(360 000, 1) dpsphp with IEEE fp16 HP,
band 1, sp 0.05, b = 1024, 2D block-cyclic; the backward-error probe on it
and on the rho = 0.999 family; then the 100-member emulation (L = 600, 601 x
1200 grid, T = 24, P = 3) from the distributed tiled factor. One JSON line on
rank 0. Usage: torchrun --nproc-per-node W tools/c5_run.py [N] [b]"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
sph._sphemu.lib().sphemu_gpu_set_device(local)
if world > 1:
    dist.init_process_group("nccl")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 360000
b = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
L = int(round(n ** 0.5))
grids = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}
P, Q = grids[world]
uid = None
if world > 1:
    obj = [sph.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
h = sph.Cholesky(n, "dpsphp", tile_size=b, hp_format="fp16", dist=(P, Q, rank, uid) if world > 1 else None)
out = {"workload": f"C5-shaped: make_spd_test_matrix({n}, 1) dpsphp/fp16 b={b} on {P}x{Q} GPUs", "n": n, "b": b,
       "gpus": world}
for rep in range(2):
    h.generate_spd(1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    h.factor()
    st = h.wait()
    dt = time.perf_counter() - t0
out["factor_device_ms_rank0"] = st.device_ms
out["factor_wall_s"] = dt
out["tflops"] = n ** 3 / 3 / dt / 1e12
out["half_saturations"] = int(st.half_saturations)
out["probe"] = h.residual_probe(1, 2)
h.generate_spd(1, rho=0.999)
h.factor()
h.wait()
out["probe_rho0999"] = h.residual_probe(1, 2, rho=0.999)
# emulation from the distributed factor
d = L * L
nt_, nphi = L + 1, 2 * L
plan = sph.ShtPlan(nt_, nphi, L)
phi = np.stack([np.full(d, x) for x in (0.6, 0.25, 0.15)])
pts = nt_ * nphi
R, T = 100, 24
mine = (R * (rank + 1)) // world - (R * rank) // world
buf = torch.empty((mine, T, nt_, nphi), dtype=torch.float64, device="cuda")
args = (plan, phi, np.zeros((T, pts)), np.ones(pts), np.full(pts, 0.04), T)
h.emulate(*args, seed=3, r_len=world, out_ptr=buf.data_ptr())
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
t0 = time.perf_counter()
h.emulate(*args, seed=3, r_len=R, out_ptr=buf.data_ptr())
torch.cuda.synchronize()
et = time.perf_counter() - t0
if world > 1:
    t = torch.tensor([et], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    et = t.item()
out["emulation"] = {"L": L, "grid": f"{nt_}x{nphi}", "replicates": R, "steps": T, "seconds": et,
                    "snapshots_per_s": R * T / et, "finite": bool(torch.isfinite(buf).all().item()),
                    "trmm_tflops": d * d * R * (30 + T) / et / 1e12}
if rank == 0:
    print(json.dumps(out), flush=True)
if world > 1:
    dist.destroy_process_group()
