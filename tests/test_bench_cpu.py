"""CPU: bench.py's host-side pieces (argument parsing, workload choice,
roofline assembly) run without a GPU, so a typo cannot surface first on the
driver's round-end run."""
import json
import os
import subprocess
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


class FakeHandle:
    def class_update_flops(self):
        return {"dp": 1e11, "sp": 1e13, "hp": 5e14}

    def flops(self):
        return {"dp": 2e11, "sp": 1.1e13, "hp": 6e14}


def phases(ms):
    names = ("potrf", "panel", "update_dp", "update_sp", "update_hp", "load")
    return {p: {"ms": ms, "launches": 1} for p in names}


def test_workload_choice():
    a = types.SimpleNamespace(workload=None)
    assert bench.pick_workload(a, 1)["n"] == 32400
    assert bench.pick_workload(a, 4)["n"] == 129600
    assert bench.GRIDS[4] == (2, 2) and bench.GRIDS[8] == (4, 2)


def test_roofline_assembly_for_both_workloads():
    for world, wl in ((1, bench.WORKLOADS["C2"]), (2, bench.WORKLOADS["C3"])):
        args = types.SimpleNamespace(sp_compute="fp16x3", world=world)
        dom = bench.roofline(FakeHandle(), wl, args, phases(10.0), 2, 50.0)
        assert dom["achieved"] > 0 and 0 < dom["frac"]
        assert dom["precision_weighted"]["t_roof_ms"] > 0
        json.dumps(dom)
        if os.path.exists(os.path.join(ROOT, "profiles", "r01_traffic.json")):
            assert dom["traffic"]["dram_bytes_per_launch"] > 0


def test_help_parses():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0 and "--gpus" in r.stdout


def test_clock_window():
    c = bench.ClockSampler(0)
    row = ["1965", "1965", "900", "0x0", "Not Active", "Not Active", "Not Active", "Active"]
    slow = ["1200", "1965", "900", "0x0", "Active", "Not Active", "Not Active", "Not Active"]
    c.rows = [(1.0, slow), (2.0, row), (2.1, row), (3.0, slow)]
    c.t0, c.t1 = 1.5, 2.5
    s = c.summary()
    assert s["sm_mhz"] == 1965.0 and s["samples"] == 2 and s["reasons"] == ["sw_power_cap"]
    c.t0, c.t1 = 2.3, 2.4  # shorter than the period: nearest row on each side
    s = c.summary()
    assert s["samples"] == 2 and "hw_slowdown" in s["reasons"]
