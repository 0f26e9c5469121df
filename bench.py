"""Benchmark of the sphemu B200 hot path (BASELINE.json configs[1] and [2]).

N = 1 (headline, configs[1] "C2"): the mixed-precision tiled Cholesky of
make_spd_test_matrix(32 400, seed 1) (L = 180, N = L^2), dpsp precision map
(band 1), 512-wide tiles; step = the dense FP64 input resident in HBM is
tiled and quantized to the precision map (mpchol.cpp:124-138,360-363), then
factored (mpchol.cpp:351-410). The N = 1 line also carries the 1-GPU point of
C3 ("c3_1gpu") so the C3 scaling curve has its base.

N > 1 (configs[2] "C3"): make_spd_test_matrix(129 600, seed 1), dpsphp with
BF16 HP storage, 2D block-cyclic over P x Q = 2x1 / 2x2 / 4x2 GPUs with copy-engine
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
# Process grids: 2D block-cyclic P x Q. With the copy-engine
# exchange and tile k+1's panel row sent first, C3 on 4 GPUs: 2x2 304 ms,
# 4x1 316 ms (tools/gpu_tasks.sh dist 4 2 / dist 4 4); 8 GPUs not measurable here.
GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}
THRESH = {"dp": 1e-12, "dpsp": 5e-6, "dpsphp": 1e-2, "dphp": 5e-2}  # acceptance_main.cpp:226


def workload_config(wl, args, world):
    """The config object both arms print (the driver compares them)."""
    grid = GRIDS.get(world, (world, 1))
    n = wl["n"]
    step = ("dense FP64 input resident in memory -> tiles at storage precision (from_dense + quantize), factor"
            if wl["input"] == "dense" else
            "make_spd_test_matrix generated into the tiles at storage precision, factor")
    return {"workload": wl["desc"], "N": n, "tile_size": wl["tile"], "variant": wl["variant"],
            "hp_format": wl["hp"], "sp_compute": args.sp_compute, "lookahead": args.lookahead,
            "parallelism": f"2D block-cyclic {grid[0]}x{grid[1]} (copy-engine panel exchange over NVLink)" if world > 1
            else "single GPU", "step": step,
            "l2": f"tiles {8 * n * n / 2 / 1e9 / world:.1f}+ GB per GPU >> 126 MB L2, no flush needed"}


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


def cpu_sht_c4_sample(t=64):
    """The oracle's SHT (ring FFT -> extended-theta FFT -> J = K I -> Wigner
    contraction, sht.cpp:226-263) at C4 (721 x 1440, L = 720) on 64 snapshots,
    all host cores: forward and inverse snapshots/s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    P = O.Plan(721, 1440, 720)
    plan_s = time.perf_counter() - t0
    c = np.stack([O.draw_random_coefficients(720, 1000 + i) for i in range(t)])
    t0 = time.perf_counter()
    f = P.inverse(c, threads=cores)
    t_inv = time.perf_counter() - t0
    t0 = time.perf_counter()
    P.forward(f, threads=cores)
    t_fwd = time.perf_counter() - t0
    return {"snapshots": t, "cores": cores, "plan_build_s": plan_s, "inverse_snapshots_per_s": t / t_inv,
            "forward_snapshots_per_s": t / t_fwd, "kind": "port (oracle restatement of sht.cpp, in-tree FFT)"}


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
    """The reference arm: the oracle's restatement of mpchol.cpp (DAG
    scheduler, all host cores, OpenBLAS tile kernels for Eigen) on this
    workload's config. The host rate keeps rising with N (more tile
    parallelism), so the K timed steps factor the workload's own N whenever
    K of them fit the time budget (C2: ~14 s each on the GPU box's host);
    otherwise (C3/C5: 134 GB+ dense) the largest sample N that fits, with the
    rate curve at 4096 / 8192 / 16384 beside it."""
    if rank != 0:
        return
    wl = pick_workload(args, world)
    for _ in range(args.warmup):
        cpu_cholesky_sample(n=2048, wl=wl)
    curve = {}
    for n in (4096, 8192, 16384):
        curve[str(n)] = cpu_cholesky_sample(n=n, wl=wl)[0]
    n_step = args.ref_n
    if not n_step:
        # estimated time of one full-size step from the 16384 rate (the rate still grows with N)
        full_t = wl["n"] ** 3 / 3 / (curve["16384"] * 1e12)
        n_step = wl["n"] if (wl["n"] <= 40000 and args.steps * full_t <= args.ref_budget_s) else 16384
    times = []
    sample = cores = None
    for _ in range(args.steps):
        _, cores, sample, t = cpu_cholesky_sample(n=n_step, wl=wl)
        times.append(t)
    v = n_step ** 3 / 3 / (sum(times) / len(times)) / 1e12
    curve[str(n_step)] = v
    same = n_step == wl["n"]
    line = {
        "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64 compute (Eigen stand-in: OpenBLAS), " + wl["variant"] + " storage",
        "data": "synthetic: make_spd_test_matrix (reference generator, bitwise)",
        "config": workload_config(wl, args, world),
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": (f"{sample}; every timed step factors the full N={wl['n']}" if same else
                                    f"{sample}; each timed step factors N={n_step} (the full N={wl['n']} dense "
                                    f"matrix does not fit the host / the time budget)")},
        "full_size": same,
        "rate_curve_tflops": curve,
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


def sp_desc(spc):
    return {"fp16x3": "fp16 hi/lo split tcgen05 (3 MMAs, fp32 accumulate)",
            "tf32x3": "3xTF32 tcgen05 (fp32 accumulate)",
            "fp64": "FP64 DMMA (the oracle's arithmetic)"}[spc]


def dominant_class(wl):
    return "sp" if wl["variant"] == "dpsp" else ("hp" if wl["variant"] in ("dpsphp", "dphp") else "dp")


def time_factor(sph, h, wl, args, world, a_dev=None, steps=None, warmup=None, clocks_index=None):
    """W untimed + K timed steps (input -> tiles at storage precision, factor),
    barrier + synchronize on both sides; max over ranks."""
    import torch
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    lib = sph._sphemu.lib()

    def step(sync=True):
        # steps are enqueued back to back (the handle orders a factorization
        # after the previous one on all of its streams); the host waits once
        # after the loop instead of idling the GPU between steps
        if a_dev is not None:
            h.load(a_dev.data_ptr(), where=sph._sphemu.DEVICE, lda=wl["n"])
        else:
            h.generate_spd(1)
        h.factor()
        return h.wait() if sync else None

    # Inside the timed region the dominant update class's launches of the
    # last timed step are bracketed by CUDA events (the roofline's achieved
    # rate): events around every launch of every step cost 2.4 ms of a 46 ms
    # C2 step (tools/step_gap.py). The full phase breakdown comes from one
    # extra profiled step afterwards.
    h.set_profiling(False)
    clocks = ClockSampler(clocks_index) if clocks_index is not None else None
    if clocks:
        clocks.__enter__()
    for w in range(warmup):
        step(sync=(w == warmup - 1))
    h.reset_phase_times()
    launches0 = lib.sphemu_gpu_launch_count()
    barrier(world)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.mark_start()
    start.record()
    for i in range(steps):
        if i == steps - 1:
            h.set_profiling(True, phases=["update_" + dominant_class(wl)])
        st = step(sync=(i == steps - 1))
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


def c1_point(sph):
    """BASELINE configs[0] (C1) end to end: the acceptance-pattern daily
    series (180 x 360, L = 45, T = 100, seed 91) -> Emulator.train(K = 2,
    period 365, P = 3, chol dp b = 256) -> emulate(100 steps, seed 42, 10
    replicates, reference RNG), on the GPU through the Python drop-in, and
    the oracle's restatement of the same pipeline on the host cores; wall
    time of each and the parity of the trained model and the fields."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    O.build()
    x = O.synth_training_series(180, 360, 45, 100, 1, 91, period=365)
    kw = dict(harmonics=2, period=365, var_order=3, band_limit=45, tile_size=256)
    sph.Emulator.train(x, **kw).emulate(100, seed=1, replicates=10)  # warm-up: module load, plans, kernels, buffers
    t0 = time.perf_counter()
    em = sph.Emulator.train(x, **kw)
    t1 = time.perf_counter()
    got = em.emulate(100, seed=42, replicates=10)
    t2 = time.perf_counter()
    cores = os.cpu_count() or 1
    m = O.train(x, 2, 365, 3, 45, "dp", 256)
    t3 = time.perf_counter()
    want = O.emulate_model(m, 100, 42, 10, threads=cores)
    t4 = time.perf_counter()
    rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
    return {"workload": "C1: 180x360 L=45 T=100 daily synthetic series (acceptance_main.cpp:535-559, seed 91); "
                        "train K=2 period 365 P=3 chol dp b=256; emulate 10 x 100 steps seed 42",
            "gpu_s": {"train": t1 - t0, "emulate": t2 - t1, "total": t2 - t0},
            "cpu_s": {"train": t3 - t2, "emulate": t4 - t3, "total": t4 - t2, "cores": cores,
                      "kind": "port (oracle restatement of pipeline.cpp/stochastic.cpp/trend.cpp)"},
            "speedup_total": (t4 - t2) / (t2 - t0),
            "parity": {"nugget_gpu": em.nugget, "nugget_cpu": m["nugget"],
                       "trend_rel": rel(em.records, m["records"]), "factor_rel": rel(em.factor(), m["v"]),
                       "fields_rel": rel(got, want), "tolerance": 1e-9},
            "api": "paper_2408_04440_b200.Emulator.train / .emulate (module.cpp:232-243 drop-in)"}


def kms_probe(h, rho=0.999):
    """Parity where the flops are: the reference generator's 0.9 decay leaves
    every tile beyond distance 1 ~0 at b >= 256, so the handle is refactored on
    the same family with rho = 0.999 (every tile O(1): 0.999^512 = 0.6) and
    probed the same way (A regenerated on the device)."""
    h.generate_spd(1, rho=rho)
    h.factor()
    h.wait()
    return {"kms_rho": rho, "kms_residual_probe": h.residual_probe(1, 2, rho=rho),
            "kms_note": "||(A - LL^T)x|| / ||Ax|| with a_ij = 0.25 d_i d_j rho^|i-j| (O(1) tiles everywhere)"}


def roofline(h, wl, args, phases, steps, ms):
    peaks = load_peaks()
    own = peaks.get("own", {})
    p_dp = own.get("fp64_dgemm_tflops", 35.5)
    f16_peak = peaks.get("bf16_tflops", 1664.2)  # kind::f16 and bf16 run at one rate
    if args.sp_compute == "fp16x3":
        p_sp = f16_peak / 3
        sp_src = "MEASURED_PEAKS.json bf16_tflops (burst; kind::f16 runs at the same rate) / 3 (3 MMAs per product)"
        sp_kernel = "k_tc_gemm<128, F16x3, UPDATE, 2> (SP-class trailing update, CTA pairs, row-scaled fp16 hi+lo)"
    else:
        p_sp = own.get("tf32x3_effective_tflops", 244.7)
        sp_src = "cuBLAS TF32 GEMM measured on this pool / 3 (profiles/peaks_r01.json)"
        sp_kernel = "k_tc_gemm<128, TF32x3, UPDATE> (SP-class trailing update)"
    if wl["hp"] == "bf16":
        p_hp, hp_src = peaks.get("bf16_tflops", 1692.6), "MEASURED_PEAKS.json bf16_tflops (burst)"
        hp_kernel = "k_tc_gemm<128, BF16, UPDATE, 2> (HP-class trailing update, CTA pairs, BF16 storage)"
    else:
        p_hp, hp_src = f16_peak, "MEASURED_PEAKS.json bf16_tflops (burst; kind::f16 runs at the same rate)"
        hp_kernel = "k_tc_gemm<128, F16, UPDATE, 2> (HP-class trailing update, CTA pairs, FP16 storage)"
    cuf = h.class_update_flops()
    bn = 256 if wl["tile"] % 256 == 0 else 128
    sp_kernel = sp_kernel.replace("<128,", f"<{bn},")
    hp_kernel = hp_kernel.replace("<128,", f"<{bn},")
    cls = {"dp": ("update_dp", p_dp, "FP64 DGEMM measured on this pool (profiles/peaks_r01.json)",
                  "k_oz_update (DP-class trailing update, INT8 tensor-core digits; DMMA for the dp variant)"),
           "sp": ("update_sp", p_sp, sp_src, sp_kernel),
           "hp": ("update_hp", p_hp, hp_src, hp_kernel)}
    dom_c = dominant_class(wl)
    ph, peak, src, kern = cls[dom_c]
    t = phases[ph]["ms"] / steps
    ach = cuf[dom_c] / (t * 1e-3) / 1e12 if t > 0 else None
    traffic = None
    for name in ("r02_traffic.json", "r01_traffic.json"):
        tf = os.path.join(ROOT, "profiles", name)
        if not os.path.exists(tf):
            continue
        tj = json.load(open(tf)).get(dom_c)
        if tj is None:
            continue
        traffic = {"dram_bytes_per_launch": tj["dram_read_bytes"] + tj["dram_write_bytes"],
                   "algorithmic_bytes_per_launch": tj["c_bytes"] + tj["panel_operand_bytes"],
                   "launch": tj["workload"] + (f", {tj['duration_us']} us alone" if "duration_us" in tj else ""),
                   "source": f"profiles/{name} (ncu --set full, one launch)"}
        if "flops" in tj and "duration_us" in tj:
            traffic["isolated_tflops"] = tj["flops"] / (tj["duration_us"] * 1e-6) / 1e12
            traffic["isolated_frac"] = traffic["isolated_tflops"] / peak
        break
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
           "peak_mma_issue": {"f16_tflops": 2229.0, "i8_tops": 4577.0,
                              "source": "profiles/r02_umma_rate.txt (tools/micro/umma_rate.cu: raw tcgen05.mma "
                                        "rate, M=128 N>=128); the SP class needs 3 f16 MMAs per product"},
           "sms": {"bulk_ctas": bulk, "device_sms": n_sm,
                   "note": "the bulk update runs on these CTAs while the POTRF/panel chain holds the rest"},
           "per_launch_basis": f"{cuf[dom_c]/1e12:.3f} TFLOP of {dom_c.upper()}-class update per step on this rank "
                               f"/ summed launch time {t:.2f} ms (CUDA events on the launching stream around each "
                               f"launch of the last timed step)"}
    fl = h.flops()
    t_roof = fl["dp"] / (p_dp * 1e12) + fl["sp"] / (p_sp * 1e12) + fl["hp"] / (p_hp * 1e12)
    world = max(1, args.world)
    dom["precision_weighted"] = {"t_roof_ms": 1e3 * t_roof / world, "frac": t_roof / world / (ms * 1e-3),
                                 "flops_split": fl, "peaks_tflops": {"dp": p_dp, "sp": p_sp, "hp": p_hp},
                                 "note": "T_roof = sum_p F_p / Peak_p over all tiles, divided by the GPU count"}
    return dom


def e2e_single(sph, wl, args, a_dev):
    """The reference-facing one-shot call (tiled_cholesky_dense's C-ABI) with
    ordinary pageable host arrays, as the drop-in callers pass them (numpy /
    std::vector): H2D of the input and D2H of the factor inside the timed
    region."""
    import ctypes as C

    import numpy as np
    import torch
    lib = sph._sphemu.lib()
    n = wl["n"]
    a_host = np.empty((n, n))
    a_host[...] = a_dev.cpu().numpy()
    f_host = np.empty((n, n))
    cfg = sph._sphemu.make_config(wl["variant"], wl["tile"], hp_format=wl["hp"], lookahead=args.lookahead,
                                  sp_compute=args.sp_compute)
    stats = sph._sphemu.CholStats()
    failed = C.c_int(-1)

    def call():
        rc = lib.sphemu_gpu_tiled_cholesky_dense(C.c_void_p(a_host.ctypes.data), 0, n, C.byref(cfg),
                                                 C.c_void_p(f_host.ctypes.data), 0, C.byref(stats), C.byref(failed))
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
    # what crosses PCIe: the lower triangle at storage width each way (FactorizationStats bytes)
    moved = int(stats.bytes_dp + stats.bytes_sp + stats.bytes_hp)
    return {"value": n ** 3 / 3 / t_e2e / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": moved,
            "d2h_bytes_per_step": moved, "ms_per_step": 1e3 * t_e2e, "steps": e2e_steps,
            "api": "sphemu_gpu_tiled_cholesky_dense (pageable host numpy arrays in and out)",
            "host_bytes_per_step": {"read": 8 * n * n, "written": 8 * n * n},
            "bytes_note": "h2d/d2h = the lower triangle at storage width (fp64 DP tiles, fp32 SP, 16-bit HP: H2D "
                          "by tile rows, D2H by tile-column groups as they finish); host threads narrow the dense "
                          "fp64 input into pinned staging and widen the factor into the caller's buffer, and "
                          "write the zeros above the diagonal"}


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


def sht_c4(sph, snapshots=1000, year_snapshots=8760):
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
    year = None
    if year_snapshots:
        # The hourly year streamed through the public API with host buffers:
        # 8 760 snapshots in calls of <= `snapshots` over one host buffer of
        # `snapshots` fields / coefficients (host RAM cannot hold the 73 GB +
        # 36 GB year twice); every call moves its inputs H2D and outputs D2H.
        import numpy as np
        h_c = np.empty((snapshots, L * L))
        h_f = np.empty((snapshots, nt, nphi))
        h_c[...] = coef.cpu().numpy()
        h_f[...] = fld.cpu().numpy()
        del coef, fld, back
        torch.cuda.empty_cache()
        plan.inverse(h_c[:8])
        plan.forward(h_f[:8])  # warm the pinned ring
        t0 = time.perf_counter()
        done = 0
        while done < year_snapshots:
            k = min(snapshots, year_snapshots - done)
            plan.inverse(h_c[:k], out=h_f[:k])
            done += k
        t_inv = time.perf_counter() - t0
        t0 = time.perf_counter()
        done = 0
        while done < year_snapshots:
            k = min(snapshots, year_snapshots - done)
            plan.forward(h_f[:k], out=h_c[:k])
            done += k
        t_fwd = time.perf_counter() - t0
        year = {"snapshots": year_snapshots, "inverse_s": t_inv, "forward_s": t_fwd,
                "inverse_snapshots_per_s": year_snapshots / t_inv, "forward_snapshots_per_s": year_snapshots / t_fwd,
                "bytes_moved_per_direction": year_snapshots * 8 * (nt * nphi + L * L),
                "api": "ShtPlan.inverse / .forward (sphemu_gpu_sht_inverse / _forward, host buffers)",
                "note": f"calls of <= {snapshots} snapshots over one pageable host buffer; chunks stream through a "
                        "ring of pinned + device slots (host copy, H2D, transform, D2H overlapped)"}
    else:
        del coef, fld, back
    del plan
    torch.cuda.empty_cache()
    return {"grid": f"{nt}x{nphi}", "band_limit": L, "snapshots": snapshots,
            "forward_snapshots_per_s": snapshots / (fwd_ms * 1e-3),
            "inverse_snapshots_per_s": snapshots / (inv_ms * 1e-3),
            "legendre_fp64_tflops_forward": flops / (fwd_ms * 1e-3) / 1e12,
            "plan_build_s": plan_s, "round_trip_rel": rt, "year": year,
            "note": "device-resident batch of 1 000 snapshots; 'year' = the 8 760-snapshot hourly year with host I/O"}


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

    peak = load_peaks().get("hbm_gbs", 6434.2)  # MEASURED_PEAKS.json is driver-written; BASELINE.md §3 value else
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


def emulation_point(sph, h, L, world=1, rank=0, replicates=100, t_out=24, order=3):
    """Emulation generator throughput (stochastic.cpp:217-277) from the
    device-resident tiled factor of handle h (d = L^2; no dense V anywhere):
    R replicates x T steps on the (L+1) x 2L grid, AR(3), device Philox
    normals, xi = V eta by the TRMM over the stored tiles, fields written to
    HBM. Distributed handles split the replicates (partial products over
    each rank's tiles reduced onto the replicate owners). Device time per
    call (CUDA events), max over ranks."""
    import numpy as np
    import torch
    d = L * L
    nt, nphi = L + 1, 2 * L
    plan = sph.ShtPlan(nt, nphi, L)
    phi = np.stack([np.full(d, x) for x in (0.6, 0.25, 0.15)[:order]])
    pts = nt * nphi
    means = np.zeros((t_out, pts))
    sigma = np.ones(pts)
    v2 = np.full(pts, 0.04)
    mine = (replicates * (rank + 1)) // world - (replicates * rank) // world
    out = torch.empty((max(1, mine), t_out, nt, nphi), dtype=torch.float64, device="cuda")
    # warm-up at the timed size: the handle's grow-only TRMM / replicate buffers
    # are allocated here, not inside the timed call (a caller generating
    # ensembles reuses them the same way)
    h.emulate(plan, phi, means, sigma, v2, t_out, seed=7, r_len=replicates, out_ptr=out.data_ptr())
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.emulate(plan, phi, means, sigma, v2, t_out, seed=7, r_len=replicates, out_ptr=out.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    dt = max_over_ranks(e0.elapsed_time(e1) * 1e-3, world)
    finite = bool(torch.isfinite(out).all().item())
    burn = 10 * order
    cols = replicates * (burn + t_out)
    del out, plan
    torch.cuda.empty_cache()
    return {"band_limit": L, "d": d, "grid": f"{nt}x{nphi}", "replicates": replicates, "steps": t_out,
            "sharding": f"replicates split over {world} GPU(s), partial TRMMs reduced over NCCL" if world > 1
            else "single GPU",
            "snapshots_per_s": replicates * t_out / dt, "seconds": dt,
            "trmm_tflops": d * d * cols / dt / 1e12,
            "trmm_note": "d^2 flops per innovation column (triangular V), R (burn + T) columns; the whole "
                         "call incl. RNG, AR(3), inverse SHT and retrend",
            "finite": finite, "api": "sphemu_gpu_emulate_chol (tiled factor, fields to HBM)"}


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
    dom = roofline(h, wl, args, h.timed_phases, 1, ms)  # the last timed step's launches
    sat = int(st.half_saturations)
    probe_kms = kms_probe(h)
    # emulation from this factor (C2: L = 180; N > 1: the C3 matrix, L = 360)
    emul = emulation_point(sph, h, int(round(n ** 0.5)), world, rank) if not args.no_emul else None
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
                "step": "generate make_spd_test_matrix tiles in place + factor", "workload": wl3["desc"],
                "parity": {"residual_probe": h3.residual_probe(1, 2), "threshold": THRESH[wl3["variant"]],
                           **kms_probe(h3)}}
        if not args.no_emul:
            c3_1["emulation"] = emulation_point(sph, h3, 360, 1, 0)
        del h3
        torch.cuda.empty_cache()

    sht = sht_throughput(sph, world)
    c4 = sht_c4(sph) if (world == 1 and not args.no_c4) else None
    side = model_side_points(sph) if (world == 1 and not args.no_c4) else None
    c1 = c1_point(sph) if (world == 1 and not args.no_c1) else None

    if rank != 0:
        return
    cpu_val, cores, sample, _ = (cpu_cholesky_sample(n=args.cpu_n, wl=wl) if not args.no_cpu
                                 else (None, 0, "skipped", 0))
    cpu_sht = cpu_sht_sample() if not args.no_cpu else (None, 0)
    if c4 is not None and not args.no_cpu:
        try:
            c4["cpu_baseline"] = cpu_sht_c4_sample()
        except Exception as e:  # noqa: BLE001 (host memory / time limits of the GPU box)
            c4["cpu_baseline"] = {"error": repr(e)[:200]}
    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": (f"f64 in/out; tiles stored per the {wl['variant']} map (DP fp64, SP fp32, HP {wl['hp']}); "
                  f"DP tiles FP64 DMMA; SP tiles {sp_desc(args.sp_compute)}; HP tiles {wl['hp']} tcgen05 "
                  f"(fp32 accumulate); panel TRSM = X B Linv^T with the FP64 inverse of the diagonal tile"),
        "data": f"synthetic: make_spd_test_matrix({n}, 1) bitwise the reference generator; SHT on random coefficients",
        "config": workload_config(wl, args, world),
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
                   "ok": bool(probe < THRESH[wl["variant"]] and probe_kms["kms_residual_probe"] < THRESH[wl["variant"]]),
                   **probe_kms,
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
    if c1:
        line["c1"] = c1
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
    ap.add_argument("--ref-n", type=int, default=0, help="reference arm step size (0: the workload's N if it fits)")
    ap.add_argument("--ref-budget-s", type=float, default=330.0, help="reference arm: time budget of the K steps")
    ap.add_argument("--cpu-n", type=int, default=16384, help="our arm's cpu_baseline sample N")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the 1-GPU C3 point on N=1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the L=720 SHT point on N=1")
    ap.add_argument("--no-emul", action="store_true", help="skip the emulation points")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 end-to-end pipeline point")
    ap.add_argument("--lookahead", type=int, default=1)
    ap.add_argument("--sp-compute", default="fp16x3", choices=["fp16x3", "tf32x3", "fp64"])
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
