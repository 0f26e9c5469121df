"""CPU, world size 2 over gloo: the host side of the multi-GPU path — every
rank derives the same 2D block-cyclic layout and panel-exchange plan
(sphemu_gpu_dist_layout, the code the device scheduler uses), tiles are
partitioned exactly, and bench.py's rank plumbing (id sharing, max over
ranks) works across processes."""
import ctypes as C
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def layout(sph, n, tile, variant, hp, P, Q, rank):
    L = sph._sphemu.lib()
    L.sphemu_gpu_dist_layout.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
    cfg = sph._sphemu.make_config(variant, tile, hp_format=hp)
    nt = (n + tile - 1) // tile
    owned = C.c_int64()
    arena = C.c_int64()
    x = np.zeros(nt * P * Q, dtype=np.int64)
    rc = L.sphemu_gpu_dist_layout(n, C.byref(cfg), P, Q, rank, C.byref(owned), C.byref(arena),
                                  C.c_void_p(x.ctypes.data))
    assert rc == 0, L.sphemu_gpu_last_error()
    return owned.value, arena.value, x.reshape(nt, P * Q)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    import paper_2408_04440_b200 as sph

    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for (P, Q) in [(2, 1), (1, 2)]:
        for variant, hp in [("dpsphp", "bf16"), ("dpsp", "fp16")]:
            owned, arena, x = layout(sph, 3000, 256, variant, hp, P, Q, rank)
            objs = [None] * world
            dist.all_gather_object(objs, (owned, arena, x.tolist()))
            out[(P, Q, variant)] = objs
    # bench plumbing: the NCCL id travels from rank 0; max over ranks
    obj = [b"uid-from-rank-0" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out["uid"] = obj[0]
    out["max"] = bench.max_over_ranks(float(rank + 1), world)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(out)


@pytest.fixture(scope="module")
def two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=240)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_tiles_partitioned_and_plans_agree(sph, two_ranks):
    nt = (3000 + 255) // 256
    for key, objs in two_ranks.items():
        if not isinstance(key, tuple):
            continue
        P, Q, variant = key
        owned = [o[0] for o in objs]
        assert sum(owned) == nt * (nt + 1) // 2, key
        # every rank derives the same exchange plan
        assert objs[0][2] == objs[1][2], key
        x = np.array(objs[0][2])
        hp = "bf16" if variant == "dpsphp" else "fp16"
        pm = sph.assign_precisions(nt, variant)
        size = lambda i, k: 256 * 256 * (8 if pm[i * (i + 1) // 2 + k] == 0 else 4 if pm[i * (i + 1) // 2 + k] == 1
                                         else 2)
        for k in range(nt - 1):
            # on 2 ranks every panel tile reaches the one rank that does not own it, if that rank reads it
            assert x[k].sum() <= sum(size(i, k) for i in range(k + 1, nt)), (key, k)
        assert x[nt - 1].sum() == 0


def _owner(i, j, P, Q):
    return i % (P * Q) if i == j else (i % P) * Q + (j % Q)


def _needers(i, k, nt, P, Q):
    need = {_owner(i, j, P, Q) for j in range(k + 1, i + 1)} | {_owner(j, i, P, Q) for j in range(i + 1, nt)}
    need.discard(_owner(i, k, P, Q))
    return need


@pytest.mark.parametrize("P,Q", [(2, 2), (4, 2), (2, 1)])
def test_exchange_plan_sends_only_to_readers(sph, P, Q):
    """Each panel tile goes point to point from its owner to the owners of row
    i and column i (P + Q ranks at most), so a rank receives ~(P + Q) / (P Q)
    of the panel bytes instead of all of them."""
    n, tile = 6000, 256
    nt = (n + tile - 1) // tile
    pm = sph.assign_precisions(nt, "dpsphp")
    size = lambda i, k: tile * tile * (8 if pm[i * (i + 1) // 2 + k] == 0 else 4 if pm[i * (i + 1) // 2 + k] == 1
                                       else 2)
    x = layout(sph, n, tile, "dpsphp", "fp16", P, Q, 0)[2]
    total = sum(size(i, k) for k in range(nt - 1) for i in range(k + 1, nt))
    for k in range(nt - 1):
        want = [0] * (P * Q)
        for i in range(k + 1, nt):
            for r in _needers(i, k, nt, P, Q):
                want[r] += size(i, k)
        assert list(x[k]) == want, k
    per_rank = x.sum(axis=0)
    assert per_rank.max() <= ((P + Q) / (P * Q) + 0.1) * total, (per_rank.max() / total)


def test_single_process_grid_2x2_partition(sph):
    nt = (3000 + 255) // 256
    owned = [layout(sph, 3000, 256, "dpsphp", "bf16", 2, 2, r)[0] for r in range(4)]
    assert sum(owned) == nt * (nt + 1) // 2 and min(owned) > 0


def test_bench_rank_plumbing(two_ranks):
    assert two_ranks["uid"] == b"uid-from-rank-0"
    assert two_ranks["max"] == 2.0


def worker8(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2408_04440_b200 as sph

    dist.init_process_group("gloo", rank=rank, world_size=world)
    owned, arena, x = layout(sph, 6000, 256, "dpsphp", "bf16", 4, 2, rank)
    objs = [None] * world
    dist.all_gather_object(objs, (owned, arena, x.tolist()))
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(objs)


def test_world8_grid_4x2_plans_agree(sph):
    """gloo world size 8: every rank of the 4 x 2 grid (C3 / C5 on 8 GPUs)
    derives the same exchange plan and the tiles partition exactly."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker8, args=(r, 8, port, q)) for r in range(8)]
    for p in ps:
        p.start()
    objs = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    nt = (6000 + 255) // 256
    assert sum(o[0] for o in objs) == nt * (nt + 1) // 2
    assert min(o[0] for o in objs) > 0
    assert all(o[2] == objs[0][2] for o in objs)
    # diagonal tiles (the FP64 band) visit every rank
    owners = {(i % 8) for i in range(nt)}
    assert owners == set(range(8))
