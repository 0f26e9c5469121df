"""Per-rank phase totals and a window of the chain/bulk timeline of the
distributed factorization (torchrun, one process per GPU)."""
import collections
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
n, b, v, hp = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
P = int(sys.argv[5]) if len(sys.argv) > 5 else world
w0 = int(sys.argv[6]) if len(sys.argv) > 6 else 100
Q = world // P
obj = [sph.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
h = sph.Cholesky(n, v, tile_size=b, hp_format=hp, dist=(P, Q, rank, obj[0]))
h.set_profiling(True)
for _ in range(2):
    h.generate_spd(1)
    h.factor()
    st = h.wait()
tl = h.timeline()
out = [f"rank {rank}: total {st.device_ms:.2f} ms"]
busy = collections.defaultdict(float)
agg = collections.defaultdict(float)
for ph, s, a, z in tl:
    busy[s] += z - a
    agg[(s, ph)] += z - a
out.append("  stream busy ms: bulk %.1f chain %.1f" % (busy[0], busy[1]))
for k, x in sorted(agg.items()):
    out.append(f"  {'bulk ' if k[0] == 0 else 'chain'} {k[1]:10s} {x:8.2f} ms")
rows = sorted(tl, key=lambda x: x[2])
span = max(z for _, _, _, z in tl)


def idle_quarters(stream):
    """Idle ms of `stream` (union of its intervals) in each quarter of the span."""
    iv = sorted((a, z) for _, s, a, z in tl if s == stream)
    res = []
    for q in range(4):
        lo, hi = span * q / 4, span * (q + 1) / 4
        cov, cur = 0.0, lo
        for a, z in iv:
            a, z = max(a, cur), min(z, hi)
            if z > a:
                cov += z - a
                cur = z
        res.append(hi - lo - cov)
    return res


out.append("  bulk  idle ms per quarter: " + " ".join("%7.2f" % x for x in idle_quarters(0)))
out.append("  chain idle ms per quarter: " + " ".join("%7.2f" % x for x in idle_quarters(1)))
for i, (ph, s, a, z) in enumerate(rows[w0:w0 + 40] if w0 >= 0 else rows[w0:]):
    out.append(f"  {'BCX'[s]} {ph:10s} {a:9.3f} {z:9.3f} {z - a:7.3f}")
for r in range(world):
    if r == rank:
        print("\n".join(out), flush=True)
    dist.barrier()
dist.destroy_process_group()
