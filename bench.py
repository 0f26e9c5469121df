"""Benchmark of the sphemu B200 hot path (BASELINE.json configs[1], "C2").

Workload C2 on one B200: the mixed-precision tiled Cholesky of
make_spd_test_matrix(32 400, seed 1) (L = 180, N = L^2) with the dpsp
precision map (band 1) and 256/512-wide tiles, plus forward+inverse SHT of
1 000 snapshots on the 181 x 360 grid at L = 180.

  step     = one factorization: the dense FP64 input (resident in HBM) is tiled
             and quantized to the precision map (mpchol.cpp:124-138,360-363),
             then factored (mpchol.cpp:351-410);
  value    = N^3/3 / device time per step, TFLOP/s (whole job, max over ranks);
  e2e      = the same through the reference-facing C-ABI call
             sphemu_gpu_tiled_cholesky_dense with pinned host buffers, H2D of
             the input and D2H of the factor inside the timed region;
  roofline = the dominant kernel (tcgen05 3xTF32 trailing update of the
             SP-class tiles) against the measured 3xTF32 rate, plus the
             precision-weighted roofline of the whole factorization;
  inputs   = 8.4 GB > 126 MB L2, so no L2 flush is needed between steps.

`--impl reference` times the reference algorithm's CPU restatement (oracle/,
the reference itself cannot be built here) on the host cores.
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

N_C2, L_C2, B_C2, VARIANT = 32400, 180, 512, "dpsp"
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
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


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
def cpu_cholesky_sample(n=8192, reps=1):
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
        O.tiled_cholesky(a, VARIANT, B_C2, workers=cores)
        best = min(best, time.perf_counter() - t0)
    return n ** 3 / 3 / best / 1e12, cores, f"make_spd_test_matrix({n}, 1), {VARIANT}, b={B_C2}; {kind_note}", best


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
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_cholesky_sample(n=4096)
    times = []
    val = sample = cores = None
    for _ in range(args.steps):
        val, cores, sample, t = cpu_cholesky_sample(n=args.ref_n)
        times.append(t)
    v = args.ref_n ** 3 / 3 / (sum(times) / len(times)) / 1e12
    line = {
        "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 compute, f32 storage (dpsp)",
        "data": "synthetic: make_spd_test_matrix (reference generator, bitwise)",
        "config": {"workload": f"C2 Cholesky bounded sample N={args.ref_n} (full C2 N={N_C2}: "
                               f"~{(N_C2/args.ref_n)**3:.0f}x the work)", "variant": VARIANT, "tile_size": B_C2},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "mixed-precision Cholesky TFLOP/s at 1/2/4/8 B200 (% of roofline); SHT snapshots/s"


# ----------------------------------------------------------------------------
# Our arm
# ----------------------------------------------------------------------------
def run_ours(args, world, rank, local):
    import ctypes as C

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    import paper_2408_04440_b200 as sph
    lib = sph._sphemu.lib()
    lib.sphemu_gpu_set_device(local)
    n, b = args.n, args.tile
    # Dense FP64 input resident in HBM (the tiled_cholesky_dense input form).
    a_dev = torch.empty((n, n), dtype=torch.float64, device="cuda")
    h = sph.Cholesky(n, VARIANT, tile_size=b, lookahead=args.lookahead, sp_compute=args.sp_compute)
    h.generate_spd(1)
    h.store(a_dev.data_ptr())          # lower triangle
    a_dev += torch.tril(a_dev, -1).T   # symmetric dense A, bitwise the reference's values
    torch.cuda.synchronize()
    fl = h.flops()
    h.set_profiling(True)

    def step():
        h.load(a_dev.data_ptr(), where=sph._sphemu.DEVICE, lda=n)
        h.factor()
        return h.wait()

    for _ in range(args.warmup):
        step()
    h.reset_phase_times()
    launches0 = lib.sphemu_gpu_launch_count()
    barrier(world)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record()
        for _ in range(args.steps):
            st = step()
        end.record()
        torch.cuda.synchronize()
    barrier(world)
    launches = lib.sphemu_gpu_launch_count() - launches0
    ms = max_over_ranks(start.elapsed_time(end) / args.steps, world)
    flops = n ** 3 / 3
    value = world * flops / (ms * 1e-3) / 1e12
    phases = h.phase_times()
    probe = h.residual_probe(1, 2)

    # Roofline: dominant kernel and whole factorization (measured peaks).
    peaks = load_peaks()
    own = peaks.get("own", {})
    p_dp = own.get("fp64_dgemm_tflops", 35.5)
    # SP class runs on the pipe of the chosen split: fp16 hi+lo (3 kind::f16
    # MMAs) -> cuBLAS FP16 / 3; 3xTF32 -> cuBLAS TF32 / 3.
    if args.sp_compute == "fp16x3":
        p_sp = own.get("fp16_tflops", 1546.6) / 3
        sp_src = "cuBLAS FP16 GEMM measured on this pool / 3 (3 kind::f16 MMAs per product; profiles/peaks_r01.json)"
        sp_kernel = "k_tc_gemm<128, F16x3, UPDATE> (SP-class trailing update, row-scaled fp16 hi+lo)"
    else:
        p_sp = own.get("tf32x3_effective_tflops", 244.7)
        sp_src = "cuBLAS TF32 GEMM measured on this pool / 3 (profiles/peaks_r01.json)"
        sp_kernel = "k_tc_gemm<128, TF32x3, UPDATE> (SP-class trailing update)"
    p_hp = peaks.get("bf16_tflops", 1692.6)
    sp_update_flops = h.class_update_flops()["sp"]
    t_sp = phases["update_sp"]["ms"] / args.steps
    dom = {"kernel": sp_kernel,
           "bound": "tensor", "achieved": sp_update_flops / (t_sp * 1e-3) / 1e12 if t_sp > 0 else None,
           "peak": p_sp, "unit": "TFLOP/s",
           "peak_source": sp_src,
           "traffic": None}
    dom["frac"] = dom["achieved"] / p_sp if dom["achieved"] else None
    t_roof = fl["dp"] / (p_dp * 1e12) + fl["sp"] / (p_sp * 1e12) + fl["hp"] / (p_hp * 1e12)
    dom["precision_weighted"] = {"t_roof_ms": 1e3 * t_roof, "frac": t_roof / (ms * 1e-3),
                                 "flops_split": fl, "peaks_tflops": {"dp": p_dp, "sp": p_sp, "hp": p_hp}}

    # End to end through the reference-facing call with pinned host buffers.
    e2e = None
    if rank == 0 or True:
        a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        a_host.copy_(a_dev)
        f_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        cfg = sph._sphemu.make_config(VARIANT, b, lookahead=args.lookahead, sp_compute=args.sp_compute)
        stats = sph._sphemu.CholStats()
        failed = C.c_int(-1)
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            rc = lib.sphemu_gpu_tiled_cholesky_dense(C.c_void_p(a_host.data_ptr()), 0, n, C.byref(cfg),
                                                     C.c_void_p(f_host.data_ptr()), 0, C.byref(stats),
                                                     C.byref(failed))
            assert rc == 0
        t_e2e = (time.perf_counter() - t0) / e2e_steps
        t_e2e = max_over_ranks(t_e2e, world)
        e2e = {"value": world * flops / t_e2e / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 8 * n * n,
               "d2h_bytes_per_step": 8 * n * n, "ms_per_step": 1e3 * t_e2e, "steps": e2e_steps,
               "api": "sphemu_gpu_tiled_cholesky_dense (host pointers, pinned)"}
        del a_host, f_host

    # SHT throughput (device-resident), forward + inverse, T = 1000 at L = 180.
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
    s0.record()
    for _ in range(reps):
        plan.inverse_device(coef.data_ptr(), SHT_T, fld.data_ptr())
        plan.forward_device(fld.data_ptr(), SHT_T, back.data_ptr())
    s1.record()
    torch.cuda.synchronize()
    sht_ms = max_over_ranks(s0.elapsed_time(s1) / reps, world)
    sht_rt = (back - coef).abs().max().item()
    sht_flops = 2 * (2 * nt * L * (L + 1)) * SHT_T
    sht = {"snapshots_per_s": world * SHT_T / (sht_ms * 1e-3), "unit": "snapshots/s (forward+inverse pair)",
           "grid": f"{nt}x{nphi}", "band_limit": L, "snapshots": SHT_T, "ms_per_batch": sht_ms,
           "legendre_fp64_tflops": sht_flops / (sht_ms * 1e-3) / 1e12, "round_trip_max_abs": sht_rt}

    if rank != 0:
        return
    cpu_val, cores, sample, _ = cpu_cholesky_sample(n=args.ref_n) if not args.no_cpu else (None, 0, "skipped", 0)
    cpu_sht = cpu_sht_sample() if not args.no_cpu else (None, 0)
    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 storage (dpsp): FP64 DMMA + 3xTF32 tcgen05",
        "data": "synthetic: make_spd_test_matrix(32400, 1) bitwise the reference generator; "
                "SHT on random coefficients",
        "config": {"workload": f"C2: tiled Cholesky N={n} (L=180) {VARIANT} b={b} + SHT 1000 snapshots "
                               f"181x360 L=180", "N": n, "tile_size": b, "variant": VARIANT,
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "inputs 8.4 GB > 126 MB L2, no flush needed"},
        "roofline": dom,
        "cpu_baseline": {"value": cpu_val, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": sample,
                         "sht_snapshots_per_s": cpu_sht[0]},
        "e2e": e2e,
        "sht": sht,
        "clocks": clk,
        "gpu_launches": int(launches),
        "phases_ms_per_step": {k: v["ms"] / args.steps for k, v in phases.items()},
        "parity": {"residual_probe": probe, "threshold": 5e-6, "ok": bool(probe < 5e-6),
                   "what": "||(A - LL^T)x|| / ||Ax|| on 2 seeded vectors, A regenerated on device; dpsp threshold "
                           "(acceptance_main.cpp:226)"},
        "half_saturations": int(st.half_saturations),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_C2)
    ap.add_argument("--tile", type=int, default=B_C2)
    ap.add_argument("--ref-n", type=int, default=8192)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--lookahead", type=int, default=1)
    ap.add_argument("--sp-compute", default="fp16x3", choices=["fp16x3", "tf32x3"])
    args = ap.parse_args()
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
