"""Benchmark of the sphemu B200 hot path (BASELINE.json configs[1] and [2]).

N = 1 (headline, configs[1] "C2"): the mixed-precision tiled Cholesky of
make_spd_test_matrix(32 400, seed 1) (L = 180, N = L^2), dpsp precision map
(band 1), 512-wide tiles; step = the dense FP64 input resident in HBM is
tiled and quantized to the precision map (mpchol.cpp:124-138,360-363), then
factored (mpchol.cpp:351-410). The N = 1 line also carries the 1-GPU point of
C3 ("c3_1gpu") so the C3 scaling curve has its base.

N > 1 (configs[2] "C3"): make_spd_test_matrix(129 600, seed 1), dpsphp with
BF16 HP storage, 2D block-cyclic over P x Q = 2x1 / 2x2 / 4x2 GPUs with NCCL
panel broadcasts; step = the generator writes each rank's owned tiles at
storage precision, then the distributed factorization. Strong scaling.

  value    = N^3/3 / device time per step, TFLOP/s (whole job, max over ranks);
  e2e      = through the public API with host buffers, H2D of the input and
             D2H of the factor inside the timed region (N = 1: the one-shot
             C-ABI call sphemu_gpu_tiled_cholesky_dense with pinned buffers;
             N > 1: the distributed handle on the C2 matrix, see e2e_dist);
  roofline = the dominant trailing-update kernel against the measured peak of
             its pipe, plus the precision-weighted roofline of the whole
             factorization;
  sht      = forward + inverse SHT of 1 000 snapshots on 181 x 360 at L = 180
             per GPU (snapshots sharded, no collective);
  inputs   = >= 8.4 GB of tiles >> 126 MB L2, so no L2 flush between steps.

`--impl reference` times the reference algorithm's CPU restatement (oracle/,
DESIGN.md §3) on the host cores on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


SHT_GRID, SHT_T = (181, 360, 180), 1000
PEAKS_FILE = os.path.join(ROOT, "profiles", "peaks_r01.json")


def load_peaks():
    peaks = {}
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        peaks.update(json.load(open(mp)))
    if os.path.exists(PEAKS_FILE):
        peaks.update({"own": json.load(open(PEAKS_FILE))})
    return peaks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region.

    nvidia-smi needs a few hundred ms to start, longer than a short timed
    region, so the sampler is started before the warm-up, waits for its first
    row, and the summary keeps only the rows stamped inside [mark_start,
    mark_end] (the nearest row on each side when the region is shorter than
    the sampling period)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 50

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.PERIOD_MS)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 10.0
            while not self.rows and time.time() < deadline and self.proc.poll() is None:
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        time.sleep(2.5 * self.PERIOD_MS / 1000.0)  # let the row after the region arrive

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def window(self):
        rows = list(self.rows)
        if self.t0 is None or self.t1 is None:
            return rows, "whole run"
        inside = [r for t, r in rows if self.t0 <= t <= self.t1]
        if inside:
            return inside, "timed region"
        before = [r for t, r in rows if t < self.t0][-1:]
        after = [r for t, r in rows if t > self.t1][:1]
        return before + after, "nearest rows around a timed region shorter than the sampling period"

    def summary(self):
        rows, where = self.window()
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows), "window": where,
                "period_ms": self.PERIOD_MS}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


# ----------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle restatement on the host cores
# ----------------------------------------------------------------------------
WORKLOADS = {
    # BASELINE.json configs[1]: the 1-GPU headline (dense FP64 input resident in HBM).
    "C2": {"n": 32400, "variant": "dpsp", "tile": 512, "hp": "fp16", "input": "dense",
           "desc": "C2: tiled Cholesky make_spd_test_matrix(32400, 1) (L=180) dpsp b=512"},
    # BASELINE.json configs[2]: 2D block-cyclic over 2/4/8 GPUs (inputs generated in place per step).
    "C3": {"n": 129600, "variant": "dpsphp", "tile": 512, "hp": "bf16", "input": "generate",
           "desc": "C3: tiled Cholesky make_spd_test_matrix(129600, 1) (L=360) dpsphp/BF16 b=512"},
}
GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}
THRESH = {"dp": 1e-12, "dpsp": 5e-6, "dpsphp": 1e-2, "dphp": 5e-2}  # acceptance_main.cpp:226


def pick_workload(args, world):
    return WORKLOADS[args.workload or ("C2" if world == 1 else "C3")]


def cpu_cholesky_sample(n=8192, reps=1, wl=None):
    wl = wl or WORKLOADS["C2"]
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    O.build()
    blas = O.find_openblas()
    kind_note = "oracle C restatement of mpchol.cpp (DAG scheduler, pthreads)"
    if blas and O.lib().so_use_blas(blas.encode()) == 0:
        kind_note += " with OpenBLAS tile kernels standing in for Eigen"
    cores = os.cpu_count() or 1
    a = O.make_spd(n, 1)
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        O.tiled_cholesky(a, wl["variant"], wl["tile"], workers=cores, hp_format=wl["hp"])
        best = min(best, time.perf_counter() - t0)
    return (n ** 3 / 3 / best / 1e12, cores,
            f"make_spd_test_matrix({n}, 1), {wl['variant']}/{wl['hp']}, b={wl['tile']}; {kind_note}", best)


def cpu_sht_sample(t=32):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O
    nt, nphi, L = SHT_GRID
    P = O.Plan(nt, nphi, L)
    c = np.stack([O.draw_random_coefficients(L, 1000 + i) for i in range(t)])
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    f = P.inverse(c, threads=cores)
    P.forward(f, threads=cores)
    dt = time.perf_counter() - t0
    return t / dt, cores


def run_reference(args, world, rank):
    if rank != 0:
        return
    wl = pick_workload(args, world)
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_cholesky_sample(n=4096, wl=wl)
    times = []
    val = sample = cores = None
    for _ in range(args.steps):
        val, cores, sample, t = cpu_cholesky_sample(n=args.ref_n, wl=wl)
        times.append(t)
    v = args.ref_n ** 3 / 3 / (sum(times) / len(times)) / 1e12
    line = {
        "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": f"f64 compute, {wl['variant']} storage",
        "data": "synthetic: make_spd_test_matrix (reference generator, bitwise)",
        "config": {"workload": f"{wl['desc']}; CPU bounded sample N={args.ref_n} "
                               f"(~{(wl['n']/args.ref_n)**3:.0f}x less work than the full N={wl['n']})",
                   "variant": wl["variant"], "tile_size": wl["tile"], "hp_format": wl["hp"]},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


METRIC = "mixed-precision Cholesky TFLOP/s at 1/2/4/8 B200 (% of roofline); SHT snapshots/s"


# ----------------------------------------------------------------------------
# Our arm
# ----------------------------------------------------------------------------
def share_uid(sph, world, rank):
    if world == 1:
        return None
    import torch.distributed as dist
    obj = [sph.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def make_handle(sph, wl, args, world, rank):
    P, Q = GRIDS.get(world, (world, 1))
    uid = share_uid(sph, world, rank)
    return sph.Cholesky(wl["n"], wl["variant"], tile_size=wl["tile"], hp_format=wl["hp"],
                        lookahead=args.lookahead, sp_compute=args.sp_compute,
                        dist=(P, Q, rank, uid) if world > 1 else None), (P, Q)


def dense_input(sph, wl):
    """The symmetric dense FP64 make_spd_test_matrix in HBM (built by a local
    1-GPU handle: generator tiles -> dense lower -> mirrored)."""
    import torch
    n = wl["n"]
    g = sph.Cholesky(n, "dp", tile_size=wl["tile"])
    g.generate_spd(1)
    a = torch.empty((n, n), dtype=torch.float64, device="cuda")
    g.store(a.data_ptr())
    del g
    a += torch.tril(a, -1).T
    torch.cuda.synchronize()
    return a


def dominant_class(wl):
    return "sp" if wl["variant"] == "dpsp" else ("hp" if wl["variant"] in ("dpsphp", "dphp") else "dp")


def time_factor(sph, h, wl, args, world, a_dev=None, steps=None, warmup=None, clocks_index=None):
    """W untimed + K timed steps (input -> tiles at storage precision, factor),
    barrier + synchronize on both sides; max over ranks."""
    import torch
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    lib = sph._sphemu.lib()

    def step():
        if a_dev is not None:
            h.load(a_dev.data_ptr(), where=sph._sphemu.DEVICE, lda=wl["n"])
        else:
            h.generate_spd(1)
        h.factor()
        return h.wait()

    # Inside the timed region only the dominant update class is bracketed by
    # CUDA events (the roofline's achieved rate); the full phase breakdown
    # comes from one extra profiled step afterwards.
    h.set_profiling(True, phases=["update_" + dominant_class(wl)])
    clocks = ClockSampler(clocks_index) if clocks_index is not None else None
    if clocks:
        clocks.__enter__()
    for _ in range(warmup):
        step()
    h.reset_phase_times()
    launches0 = lib.sphemu_gpu_launch_count()
    barrier(world)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.mark_start()
    start.record()
    for _ in range(steps):
        st = step()
    end.record()
    torch.cuda.synchronize()
    if clocks:
        clocks.mark_end()
        clocks.__exit__()
    barrier(world)
    launches = lib.sphemu_gpu_launch_count() - launches0
    ms = max_over_ranks(start.elapsed_time(end) / steps, world)
    h.timed_phases = h.phase_times()
    h.set_profiling(True)
    h.reset_phase_times()
    step()
    h.all_phases = h.phase_times()
    h.set_profiling(False)
    return ms, st, launches, clocks


def roofline(h, wl, args, phases, steps, ms):
    peaks = load_peaks()
    own = peaks.get("own", {})
    p_dp = own.get("fp64_dgemm_tflops", 35.5)
    if args.sp_compute == "fp16x3":
        p_sp = own.get("fp16_tflops", 1546.6) / 3
        sp_src = "cuBLAS FP16 GEMM measured on this pool / 3 (3 kind::f16 MMAs per product; profiles/peaks_r01.json)"
        sp_kernel = "k_tc_gemm<128, F16x3, UPDATE, 1> (SP-class trailing update, row-scaled fp16 hi+lo)"
    else:
        p_sp = own.get("tf32x3_effective_tflops", 244.7)
        sp_src = "cuBLAS TF32 GEMM measured on this pool / 3 (profiles/peaks_r01.json)"
        sp_kernel = "k_tc_gemm<128, TF32x3, UPDATE> (SP-class trailing update)"
    if wl["hp"] == "bf16":
        p_hp, hp_src = peaks.get("bf16_tflops", 1692.6), "MEASURED_PEAKS.json bf16_tflops (burst)"
        hp_kernel = "k_tc_gemm<128, BF16, UPDATE, 2> (HP-class trailing update, CTA pairs, BF16 storage)"
    else:
        p_hp, hp_src = own.get("fp16_tflops", 1546.6), "cuBLAS FP16 GEMM measured on this pool (profiles/peaks_r01.json)"
        hp_kernel = "k_tc_gemm<128, F16, UPDATE, 2> (HP-class trailing update, CTA pairs, FP16 storage)"
    cuf = h.class_update_flops()
    bn = 256 if wl["tile"] % 256 == 0 else 128
    sp_kernel = sp_kernel.replace("<128,", f"<{bn},")
    hp_kernel = hp_kernel.replace("<128,", f"<{bn},")
    cls = {"dp": ("update_dp", p_dp, "FP64 DGEMM measured on this pool (profiles/peaks_r01.json)",
                  "k_update_fp64_v2 (DP-class trailing update, DMMA)"),
           "sp": ("update_sp", p_sp, sp_src, sp_kernel),
           "hp": ("update_hp", p_hp, hp_src, hp_kernel)}
    dom_c = dominant_class(wl)
    ph, peak, src, kern = cls[dom_c]
    t = phases[ph]["ms"] / steps
    ach = cuf[dom_c] / (t * 1e-3) / 1e12 if t > 0 else None
    traffic = None
    tf = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tf) and dom_c in ("sp", "hp"):
        tj = json.load(open(tf))[dom_c]
        traffic = {"dram_bytes_per_launch": tj["dram_read_bytes"] + tj["dram_write_bytes"],
                   "algorithmic_bytes_per_launch": tj["c_bytes"] + tj["panel_operand_bytes"],
                   "launch": f"{tj['workload']}: {tj['sub_tiles']} sub-tiles of 128x256, K=512",
                   "source": "profiles/r01_traffic.json (ncu --set full, one launch)"}
    # The bulk update runs on SMs - reserve CTAs (the reserve serves the
    # POTRF/panel chain stream concurrently); frac is against the whole GPU.
    import torch
    n_sm = (torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            if torch.cuda.is_available() else 148)
    # one GPU: 8 SMs reserved for the chain except in the last 32 steps (32); multi-GPU: 32 (2 GPUs) or 48
    world = max(1, args.world)
    bulk = [n_sm - 8, n_sm - 32] if world == 1 else [n_sm - (32 if world < 4 else 48)]
    dom = {"kernel": kern, "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
           "frac": ach / peak if ach else None, "peak_source": src, "traffic": traffic,
           "sms": {"bulk_ctas": bulk, "device_sms": n_sm,
                   "note": "the bulk update runs on these CTAs while the POTRF/panel chain holds the rest"},
           "per_launch_basis": f"{cuf[dom_c]/1e12:.3f} TFLOP of {dom_c.upper()}-class update per step on this rank "
                               f"/ summed launch time {t:.2f} ms (CUDA events on the launching stream)"}
    fl = h.flops()
    t_roof = fl["dp"] / (p_dp * 1e12) + fl["sp"] / (p_sp * 1e12) + fl["hp"] / (p_hp * 1e12)
    world = max(1, args.world)
    dom["precision_weighted"] = {"t_roof_ms": 1e3 * t_roof / world, "frac": t_roof / world / (ms * 1e-3),
                                 "flops_split": fl, "peaks_tflops": {"dp": p_dp, "sp": p_sp, "hp": p_hp},
                                 "note": "T_roof = sum_p F_p / Peak_p over all tiles, divided by the GPU count"}
    return dom


def e2e_single(sph, wl, args, a_dev):
    """The reference-facing one-shot call with pinned host buffers: H2D of the
    input and D2H of the factor inside the timed region."""
    import ctypes as C
    import torch
    lib = sph._sphemu.lib()
    n = wl["n"]
    a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    a_host.copy_(a_dev)
    f_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    cfg = sph._sphemu.make_config(wl["variant"], wl["tile"], hp_format=wl["hp"], lookahead=args.lookahead,
                                  sp_compute=args.sp_compute)
    stats = sph._sphemu.CholStats()
    failed = C.c_int(-1)

    def call():
        rc = lib.sphemu_gpu_tiled_cholesky_dense(C.c_void_p(a_host.data_ptr()), 0, n, C.byref(cfg),
                                                 C.c_void_p(f_host.data_ptr()), 0, C.byref(stats), C.byref(failed))
        assert rc == 0, rc

    for _ in range(max(3, args.warmup)):
        call()  # warm-up: first-call module load, the handle cache, first touch of the host staging pool
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        call()
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    lib.sphemu_gpu_release_cache()
    del a_host, f_host
    return {"value": n ** 3 / 3 / t_e2e / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 8 * n * n,
            "d2h_bytes_per_step": 8 * n * n, "ms_per_step": 1e3 * t_e2e, "steps": e2e_steps,
            "api": "sphemu_gpu_tiled_cholesky_dense (host pointers, pinned)",
            "bytes_note": "counted as the dense n x n in and out; the library moves the lower triangle at storage "
                          "width (fp64 DP tiles, fp32 the rest: H2D by tile rows, D2H by tile-column groups as they "
                          "finish), host threads narrow / widen it and stream the zeros"}


def e2e_dist(sph, args, world, rank):
    """N GPUs through the distributed handle with host buffers: the dense C2
    input lives once in shared host memory (/dev/shm, registered with every
    rank's CUDA context), each rank copies the rows it owns; the factor is
    gathered over NCCL and written to rank 0's pinned host buffer."""
    import ctypes as C
    import torch
    wl = WORKLOADS["C2"]
    n = wl["n"]
    path = f"/dev/shm/sphemu_bench_{os.environ.get('MASTER_PORT', '0')}"
    if rank == 0:
        a_dev = dense_input(sph, wl)
        a_host = torch.from_file(path, shared=True, size=n * n, dtype=torch.float64).view(n, n)
        a_host.copy_(a_dev)
        del a_dev
        torch.cuda.empty_cache()
    barrier(world)
    if rank != 0:
        a_host = torch.from_file(path, shared=True, size=n * n, dtype=torch.float64).view(n, n)
    cudart = torch.cuda.cudart()
    registered = int(cudart.cudaHostRegister(a_host.data_ptr(), 8 * n * n, 0)) == 0
    f_host = torch.empty((n, n) if rank == 0 else (1, 1), dtype=torch.float64, pin_memory=True)
    h, grid = make_handle(sph, wl, args, world, rank)
    lib = sph._sphemu.lib()

    def call():
        h.load(a_host.numpy())
        h.factor()
        h.wait()
        rc = lib.sphemu_gpu_chol_store_dense(h.h, C.c_void_p(f_host.data_ptr()), 0, n)
        assert rc == 0, rc

    call()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        call()
    t_e2e = max_over_ranks((time.perf_counter() - t0) / e2e_steps, world)
    del h
    if registered:
        cudart.cudaHostUnregister(a_host.data_ptr())
    barrier(world)
    if rank == 0:
        os.unlink(path)
    return {"value": n ** 3 / 3 / t_e2e / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 8 * n * n,
            "d2h_bytes_per_step": 8 * n * n, "ms_per_step": 1e3 * t_e2e, "steps": e2e_steps,
            "workload": f"{wl['desc']} over {grid[0]}x{grid[1]} GPUs (C3's 134 GB dense host input and output "
                        f"exceed this box's 196 GB host RAM)",
            "api": "Cholesky(dist=...).load(host) + factor + sphemu_gpu_chol_store_dense(host); input in "
                   "shared host memory" + (" (registered)" if registered else " (pageable)")}


def sht_throughput(sph, world):
    import torch
    nt, nphi, L = SHT_GRID
    plan = sph.ShtPlan(nt, nphi, L)
    coef = torch.randn(SHT_T, L * L, dtype=torch.float64, device="cuda")
    fld = torch.empty(SHT_T, nt, nphi, dtype=torch.float64, device="cuda")
    back = torch.empty_like(coef)
    for _ in range(2):
        plan.inverse_device(coef.data_ptr(), SHT_T, fld.data_ptr())
        plan.forward_device(fld.data_ptr(), SHT_T, back.data_ptr())
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    barrier(world)
    s0.record()
    for _ in range(reps):
        plan.inverse_device(coef.data_ptr(), SHT_T, fld.data_ptr())
        plan.forward_device(fld.data_ptr(), SHT_T, back.data_ptr())
    s1.record()
    torch.cuda.synchronize()
    sht_ms = max_over_ranks(s0.elapsed_time(s1) / reps, world)
    sht_rt = (back - coef).abs().max().item()
    sht_flops = 2 * (2 * nt * L * (L + 1)) * SHT_T
    return {"snapshots_per_s": world * SHT_T / (sht_ms * 1e-3), "unit": "snapshots/s (forward+inverse pair)",
            "grid": f"{nt}x{nphi}", "band_limit": L, "snapshots_per_gpu": SHT_T, "ms_per_batch": sht_ms,
            "sharding": "snapshots sharded across GPUs, no collective" if world > 1 else "single GPU",
            "legendre_fp64_tflops_per_gpu": sht_flops / (sht_ms * 1e-3) / 1e12, "round_trip_max_abs": sht_rt}


def sht_c4(sph, snapshots=1000):
    """BASELINE configs[3] (C4): 721 x 1440 grid (720 x 1440 cannot resolve L = 720), L = 720,
    forward and inverse timed separately on a device-resident batch."""
    import torch
    nt, nphi, L = 721, 1440, 720
    t0 = time.perf_counter()
    plan = sph.ShtPlan(nt, nphi, L, wigner_cap_bytes=8 << 30)  # the reference's 2 GiB cap rejects L = 720 (F5)
    plan_s = time.perf_counter() - t0
    coef = torch.randn(snapshots, L * L, dtype=torch.float64, device="cuda")
    fld = torch.empty(snapshots, nt, nphi, dtype=torch.float64, device="cuda")
    back = torch.empty_like(coef)
    plan.inverse_device(coef.data_ptr(), snapshots, fld.data_ptr())
    plan.forward_device(fld.data_ptr(), snapshots, back.data_ptr())
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    plan.inverse_device(coef.data_ptr(), snapshots, fld.data_ptr())
    ev[1].record()
    plan.forward_device(fld.data_ptr(), snapshots, back.data_ptr())
    ev[2].record()
    torch.cuda.synchronize()
    inv_ms, fwd_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    flops = 2 * nt * L * (L + 1) * snapshots
    rt = ((back - coef).abs().max() / coef.abs().max()).item()
    del coef, fld, back, plan
    torch.cuda.empty_cache()
    return {"grid": f"{nt}x{nphi}", "band_limit": L, "snapshots": snapshots,
            "forward_snapshots_per_s": snapshots / (fwd_ms * 1e-3),
            "inverse_snapshots_per_s": snapshots / (inv_ms * 1e-3),
            "legendre_fp64_tflops_forward": flops / (fwd_ms * 1e-3) / 1e12,
            "plan_build_s": plan_s, "round_trip_rel": rt,
            "note": "the driver's 8 760-snapshot hourly year runs in chunks of this batch"}


def model_side_points(sph):
    """The §8f rows either side of the factorization, device-resident through
    the C-ABI, kernel-only time from CUDA events on the default stream:
    fit_var at the C2 size (d = 32 400, T = 1 000, order 3) and retrend on the
    C4 grid (721 x 1440, K = 5, 4 x 96 fields). Algorithmic HBM GB/s against
    MEASURED_PEAKS.json."""
    import ctypes as C

    import numpy as np
    import torch
    lib = sph._sphemu.lib()
    vp = C.c_void_p
    out = {}
    T, d, order = 1000, 180 * 180, 3
    c = torch.cumsum(torch.randn(1, T, d, dtype=torch.float64, device="cuda") * 0.05, dim=1)
    res = torch.empty(T - order, d, dtype=torch.float64, device="cuda")
    phi = np.empty(order * d)
    se = np.empty(order * d)
    zc, uc, nrm = C.c_int64(), C.c_int64(), C.c_double()

    def fv():
        assert lib.sphemu_gpu_fit_var(vp(c.data_ptr()), 1, 1, T, d, order, vp(phi.ctypes.data),
                                      vp(se.ctypes.data), vp(res.data_ptr()), 1, C.byref(zc), C.byref(uc),
                                      C.byref(nrm)) == 0

    points, K, R, Tt = 721 * 1440, 5, 4, 96
    rec = np.random.default_rng(1).standard_normal((points, 5 + 2 * K))
    rec[:, -1] = 1.0 + np.abs(rec[:, -1])
    z = torch.randn(R, Tt, points, dtype=torch.float64, device="cuda")
    y = torch.empty_like(z)
    rec_d = torch.from_numpy(rec).cuda()  # device-resident records: read in place by the kernel

    def rt():
        assert lib.sphemu_gpu_retrend(vp(z.data_ptr()), 1, R, Tt, vp(rec_d.data_ptr()), points, K, 8760, None, 0,
                                      None, 0, 1, vp(y.data_ptr()), 1) == 0

    peak = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")))["hbm_gbs"]
    for name, fn, nbytes, what in (
            ("fit_var", fv, 16 * T * d + 8 * (T - order) * d, "C2 size: d=32400, T=1000, order 3 (series read "
             "twice + residuals written)"),
            ("retrend", rt, 16 * R * Tt * points, "C4 grid 721x1440, K=5, 4x96 fields (z read + y written)")):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(5):
            fn()
        s1.record()
        torch.cuda.synchronize()
        ms = s0.elapsed_time(s1) / 5
        out[name] = {"ms_per_call": ms, "algorithmic_gbs_per_call": nbytes / ms / 1e6, "hbm_peak_gbs": peak,
                     "workload": what, "note": "per C-ABI call incl. its small host transfers; the kernel-only "
                                               "figures are in profiles/r01_ncu_fit_var.txt / r01_ncu_trend.txt"}
    del c, res, z, y, rec_d
    torch.cuda.empty_cache()
    return out


def emulation_point(sph, L=90, replicates=100, t_out=24, order=3, world=1, rank=0):
    """Emulation generator throughput (stochastic.cpp:217-277): R replicates x T steps on the (L+1) x 2L grid,
    V = the device factor of make_spd_test_matrix(L^2) (dp), AR(3), device Philox normals; the one-shot C-ABI
    call with host buffers (V in, fields out) is the timed unit."""
    import numpy as np
    d = L * L
    h = sph.Cholesky(d, "dp", tile_size=256)
    h.generate_spd(1)
    h.factor()
    h.wait()
    v = h.factor_dense()
    del h
    nt, nphi = L + 1, 2 * L
    plan = sph.ShtPlan(nt, nphi, L)
    phi = np.stack([np.full(d, x) for x in (0.6, 0.25, 0.15)[:order]])
    pts = nt * nphi
    means = np.zeros((t_out, pts))
    sigma = np.ones(pts)
    v2 = np.full(pts, 0.04)
    sph._sphemu.emulate(plan, v, phi, means, sigma, v2, t_out, 7, 2, "philox")  # warm-up
    # replicates sharded over the ranks (draws depend only on the replicate: no communication)
    per = (replicates + world - 1) // world
    r0 = min(replicates, rank * per)
    cnt = max(0, min(per, replicates - r0))
    barrier(world)
    t0 = time.perf_counter()
    out = sph._sphemu.emulate(plan, v, phi, means, sigma, v2, t_out, 7, cnt, "philox", r_begin=r0) if cnt else \
        np.zeros(1)
    dt = max_over_ranks(time.perf_counter() - t0, world)
    burn = 10 * order
    return {"band_limit": L, "d": d, "grid": f"{nt}x{nphi}", "replicates": replicates, "steps": t_out,
            "sharding": f"replicate ranges over {world} GPU(s)",
            "snapshots_per_s": replicates * t_out / dt, "seconds": dt,
            "trmm_fp64_tflops": d * d * replicates * (burn + t_out) / dt / 1e12,
            "finite": bool(np.isfinite(out).all()),
            "api": "sphemu_gpu_emulate (host V and fields, H2D/D2H inside)"}


def run_ours(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    import paper_2408_04440_b200 as sph
    lib = sph._sphemu.lib()
    lib.sphemu_gpu_set_device(local)
    args.world = world
    wl = pick_workload(args, world)
    n = wl["n"]
    a_dev = dense_input(sph, wl) if wl["input"] == "dense" else None
    h, grid = make_handle(sph, wl, args, world, rank)
    h.set_profiling(True)
    ms, st, launches, clocks = time_factor(sph, h, wl, args, world, a_dev=a_dev, clocks_index=local)
    flops = n ** 3 / 3
    value = flops / (ms * 1e-3) / 1e12
    phases = h.all_phases
    probe = h.residual_probe(1, 2)
    dom = roofline(h, wl, args, h.timed_phases, args.steps, ms)
    sat = int(st.half_saturations)
    del h
    torch.cuda.empty_cache()

    if world == 1:
        e2e = e2e_single(sph, wl, args, a_dev) if a_dev is not None else None
    else:
        e2e = e2e_dist(sph, args, world, rank) if not args.no_e2e else None
    del a_dev
    torch.cuda.empty_cache()

    # C3 on one GPU (the 1-GPU point of the C3 scaling curve; the headline N=1 line is C2).
    c3_1 = None
    if world == 1 and not args.no_c3:
        wl3 = WORKLOADS["C3"]
        h3, _ = make_handle(sph, wl3, args, 1, 0)
        ms3, _, _, _ = time_factor(sph, h3, wl3, args, 1, steps=2, warmup=1)
        c3_1 = {"ms_per_step": ms3, "tflops": wl3["n"] ** 3 / 3 / (ms3 * 1e-3) / 1e12, "steps": 2, "warmup": 1,
                "step": "generate make_spd_test_matrix tiles in place + factor", "workload": wl3["desc"]}
        del h3
        torch.cuda.empty_cache()

    sht = sht_throughput(sph, world)
    c4 = sht_c4(sph) if (world == 1 and not args.no_c4) else None
    emul = emulation_point(sph, world=world, rank=rank) if not args.no_c4 else None
    side = model_side_points(sph) if (world == 1 and not args.no_c4) else None

    if rank != 0:
        return
    cpu_val, cores, sample, _ = (cpu_cholesky_sample(n=args.ref_n, wl=wl) if not args.no_cpu
                                 else (None, 0, "skipped", 0))
    cpu_sht = cpu_sht_sample() if not args.no_cpu else (None, 0)
    clk = clocks.summary()
    step_desc = ("dense FP64 input resident in HBM -> tiles at storage precision (from_dense + quantize), factor"
                 if wl["input"] == "dense" else
                 "make_spd_test_matrix generated into the owned tiles at storage precision, factor")
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": (f"f64 compute semantics; storage {wl['variant']} ({wl['hp']} HP): FP64 DMMA, "
                  f"{args.sp_compute} tcgen05 for SP, {wl['hp']} tcgen05 for HP"),
        "data": f"synthetic: make_spd_test_matrix({n}, 1) bitwise the reference generator; SHT on random coefficients",
        "config": {"workload": f"{wl['desc']} + SHT 1000 snapshots 181x360 L=180 per GPU", "N": n,
                   "tile_size": wl["tile"], "variant": wl["variant"], "hp_format": wl["hp"],
                   "sp_compute": args.sp_compute, "lookahead": args.lookahead,
                   "parallelism": f"2D block-cyclic {grid[0]}x{grid[1]} (NCCL panel broadcasts)" if world > 1
                   else "single GPU",
                   "step": step_desc,
                   "l2": f"tiles {8 * n * n / 2 / 1e9 / world:.1f}+ GB per GPU >> 126 MB L2, no flush needed"},
        "roofline": dom,
        "cpu_baseline": {"value": cpu_val, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": sample, "sht_snapshots_per_s": cpu_sht[0]},
        "e2e": e2e,
        "sht": sht,
        "clocks": clk,
        "gpu_launches": int(launches),
        "phases_ms_per_step_rank0": {k: v["ms"] for k, v in phases.items()},
        "phases_note": "one extra fully profiled step after the timed region (busy time per phase, chain and bulk "
                       "streams overlap)",
        "parity": {"residual_probe": probe, "threshold": THRESH[wl["variant"]],
                   "ok": bool(probe < THRESH[wl["variant"]]),
                   "what": "||(A - LL^T)x|| / ||Ax|| on 2 seeded vectors, A regenerated on device; thresholds of "
                           "acceptance_main.cpp:226"},
        "half_saturations": sat,
    }
    if c3_1:
        line["c3_1gpu"] = c3_1
    if c4:
        line["sht_c4"] = c4
    if emul:
        line["emulation"] = emul
    if side:
        line["model_side"] = side
    emit(line)


_JSON_OUT = None


def emit(line):
    """The one JSON line, on the process's original stdout. Everything else
    that native code writes to fd 1 (NCCL's version banner, library chatter)
    is routed to stderr by main() so stdout carries exactly this line."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: C2 on 1 GPU, C3 (2D block-cyclic) on more")
    ap.add_argument("--ref-n", type=int, default=8192)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the 1-GPU C3 point on N=1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the L=720 SHT point on N=1")
    ap.add_argument("--lookahead", type=int, default=1)
    ap.add_argument("--sp-compute", default="fp16x3", choices=["fp16x3", "tf32x3"])
    args = ap.parse_args()
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
