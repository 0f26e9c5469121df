"""torchrun worker for tests/test_gpu_dist.py (one process per GPU): the 2D
block-cyclic factor with point-to-point panel exchange must equal the
single-GPU factor bitwise (same per-tile operations in the same k order) on
grids 1xW and Wx1 (and 2x2 at W = 4), on the reference generator and on its
non-decaying rho = 0.999 form; the distributed emulation (partial TRMMs over
each rank's tiles reduced onto the replicate owners) must match the 1-GPU
emulation; prints one line per check, "FAIL" on a mismatch."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2408_04440_b200 as sph  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
sph._sphemu.lib().sphemu_gpu_set_device(local)
dist.init_process_group("nccl")
grids = [(1, world), (world, 1)] + ([(2, 2)] if world == 4 else []) + ([(4, 2)] if world == 8 else [])
ok = True


def uid():
    obj = [sph.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


for n, b, v, hp, rho in ((3000, 256, "dpsphp", "fp16", None), (3000, 256, "dpsphp", "bf16", 0.999),
                         (4100, 512, "dpsp", "fp16", 0.999)):
    ref = None
    if rank == 0:
        h1 = sph.Cholesky(n, v, tile_size=b, hp_format=hp)
        h1.generate_spd(3, rho=rho)
        h1.factor()
        h1.wait()
        ref = h1.factor_dense()
        del h1
    for P, Q in grids:
        h = sph.Cholesky(n, v, tile_size=b, hp_format=hp, dist=(P, Q, rank, uid()))
        h.generate_spd(3, rho=rho)
        h.factor()
        h.wait()
        probe = h.residual_probe(3, 2, rho=rho)
        f = h.factor_dense()
        if rank == 0:
            same = np.array_equal(f, ref)
            ok &= same
            print(f"{'ok' if same else 'FAIL'} factor n={n} b={b} {v}/{hp} rho={rho} grid {P}x{Q} "
                  f"probe={probe:.2e}", flush=True)
        del h

# distributed emulation vs one GPU (Philox stream: draws depend only on the replicate)
Lb, t_out, R = 40, 6, 5
d = Lb * Lb
nt_, nphi = Lb + 1, 2 * Lb
plan = sph.ShtPlan(nt_, nphi, Lb)
phi = np.stack([np.full(d, x) for x in (0.5, 0.2)])
rng = np.random.default_rng(1)
sigma = 0.5 + rng.random(nt_ * nphi)
v2 = np.full(nt_ * nphi, 0.04)
means = np.zeros((t_out, nt_ * nphi))
full = None
if rank == 0:
    h1 = sph.Cholesky(d, "dpsphp", tile_size=256)
    h1.generate_spd(5, rho=0.999)
    h1.factor()
    h1.wait()
    full = h1.emulate(plan, phi, means, sigma, v2, t_out, seed=4, r_len=R)
    del h1
for P, Q in grids[:1]:
    h = sph.Cholesky(d, "dpsphp", tile_size=256, dist=(P, Q, rank, uid()))
    h.generate_spd(5, rho=0.999)
    h.factor()
    h.wait()
    mine = h.emulate(plan, phi, means, sigma, v2, t_out, seed=4, r_len=R)
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        got = np.concatenate(parts)
        err = np.abs(got - full).max() / np.abs(full).max()
        good = got.shape == full.shape and err < 1e-5
        ok &= good
        print(f"{'ok' if good else 'FAIL'} emulate grid {P}x{Q} rel err {err:.2e}", flush=True)
    del h
if rank == 0:
    print("ALL OK" if ok else "SOME FAILED", flush=True)
dist.destroy_process_group()
