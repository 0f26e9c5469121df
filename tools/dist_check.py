"""Multi-GPU 2D block-cyclic Cholesky check (run under torchrun, one process
per GPU): the gathered distributed factor must equal the single-GPU factor
bitwise (same per-tile operations in the same k order), plus timing."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_04440_b200 as sph  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
sph._sphemu.lib().sphemu_gpu_set_device(local)
dist.init_process_group("nccl")
grids = [(1, world), (world, 1)] if world > 1 else [(1, 1)]
if world == 4:
    grids.append((2, 2))
for n, b, v in ((3000, 256, "dpsphp"), (8192, 512, "dpsp")):
    ref = None
    if rank == 0:
        h1 = sph.Cholesky(n, v, tile_size=b, lookahead=0)
        h1.generate_spd(3)
        h1.factor()
        h1.wait()
        ref = h1.factor_dense()
        del h1
    for P, Q in grids:
        obj = [sph.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        h = sph.Cholesky(n, v, tile_size=b, lookahead=int(os.environ.get("LOOKAHEAD", "1")), dist=(P, Q, rank, obj[0]))
        h.generate_spd(3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.factor()
        st = h.wait()
        dt = time.perf_counter() - t0
        probe = h.residual_probe(3, 2)
        f = h.factor_dense()
        if rank == 0:
            same = np.array_equal(f, ref)
            print(f"n={n} b={b} {v} grid {P}x{Q}: bitwise-equal-to-1GPU={same} maxdiff={np.abs(f - ref).max():.3e} "
                  f"probe={probe:.3e} {st.device_ms:.1f} ms dev, {dt*1e3:.1f} ms wall", flush=True)
        del h
dist.destroy_process_group()
