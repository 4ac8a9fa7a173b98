#!/usr/bin/env python
"""bench.py — fp64 cell-updates/s of the explicit-implicit splitting hot path on B200.

Default workload: BASELINE.json configs[4] (C5), one 2^27-cell grid with 4096-cell random
segments (~14.5k cavitation bubbles), 500 large steps: the largest single-GPU configuration and
the one the metric's 1/2/4/8-GPU scaling is quoted on (domain decomposition).  One bench
"step" = one large time step of the whole method over the whole
grid: the tiled fast pass, the window / whole-tile full steps, the next dt.  The K timed steps
start from the seeded initial state (so they include the creation step); the state (2 GB) is
resident in HBM and larger than the 126 MB L2.

--workload C3: BASELINE configs[2], the batched cavitation ensemble (65,536 grids of N=1024,
2000 steps) as ONE launch of the member-resident kernel (eis_step(K)); --workload C4: BASELINE
configs[3] (16,384 grids of N=4096), tiled layout through EIS_LAYOUT_AUTO (three launches per
step plus the per-member finish).  --mode selects the implicit-region treatment (default: the
paper's dual time stepping).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl eis|reference] [--workload C3|C4|C1|C2|C5]
                  [--mode 0|1|2|3]

Multi-GPU (torchrun): C5 cuts the grid into tile-aligned rank slices: per step the local
kernels, a 10-cell halo exchange with the neighbour ranks and an all-reduce(MIN) of the CFL pair
(paper_2211_00705_b200.decomp); C3/C4 interleave members over ranks with no collective in the
data path.  Scaling "strong" (the problem is fixed); timing is the max over ranks.
--impl reference times the CPU oracle (oracle/, OpenMP over the host cores) on a bounded sample (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic fp64 operations per cell-update of the bulk path, SURVEY §8(d)'s count (a division
# = 1 op): u = m/rho 1, p 2, HLL flux of one edge per cell ~17 (Davis speeds, the two physical
# fluxes, the intermediate state), update 6.  (The kernel executes more: rcp refinement, the
# creation pre-filter, the CFL partials; those are not algorithmic work.)
FLOP_PER_CELL_UPDATE = 26
C5_BYTES_PER_CELL_UPDATE = 32  # the fast pass: read rho, mom; write rho, mom (fp64; widths of
                                # tiles whose widths are all h_av are neither read nor written)
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: SMs x FP64 FMA/clk x 2 x max clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default 2000 (C3/C4), 500 (C5)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="eis", choices=["eis", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C5", "C3", "C4", "C1", "C2"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--members", type=int, default=0, help="profiling only: fewer ensemble members")
    ap.add_argument("--start-steps", type=int, default=0, help="profiling only: untimed steps before the timed launch")
    ap.add_argument("--mode", type=int, default=None, choices=[0, 1, 2, 3],
                    help="implicit-region treatment: 0 split/DTS (default, the paper), 1 explicit, 2 LTS, 3 Newton")
    a = ap.parse_args()
    global MODE
    MODE = a.mode
    if a.steps is None:
        a.steps = 500 if a.workload == "C5" else 2000
    return a


MODE = None  # --mode: the implicit-region treatment (default: the workload's, SPLIT = the paper's DTS)
MODE_NAMES = {0: "split (dual time stepping)", 1: "explicit", 2: "local time stepping", 3: "newton (chord Newton)"}


def with_mode(w):
    if MODE is not None:
        w["params"] = dict(w["params"])
        w["params"]["mode"] = MODE
    return w


def workload(name, members=None):
    from paper_2211_00705_b200 import workloads as W
    if name == "C3":
        return with_mode(W.c3(members=members) if members is not None else W.c3())
    if name == "C4":
        return with_mode(W.c4(members=members) if members is not None else W.c4())
    if name == "C1":
        return with_mode(W.c1())
    if name == "C5":
        return with_mode(W.c5(n_cells=members) if members is not None else W.c5())
    return with_mode(W.c2())


def total_members(name):
    return {"C3": 65536, "C4": 16384, "C1": 1, "C2": 1}[name]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        if not self.rows:  # region shorter than one period: one sample right after
            out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i",
                                  str(self.device)], capture_output=True, text=True).stdout
            self.rows = [[s.strip() for s in out.strip().split(",")]] if out.strip() else []
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def job_rates(dist, torch, world, st, ms):
    """DTS iterations/s and interface solves/s of the whole job (the paper's "local
    iterations"), and simulated time per wall-second (the timed steps start at t = 0)."""
    n = [int(st["dts_iters"]), int(st["iface_solves"])]
    if world > 1:
        c = torch.tensor(n, device="cuda", dtype=torch.int64)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        n = [int(x) for x in c.tolist()]
    sec = ms * 1e-3
    return {"dts_iters_per_s": n[0] / sec, "iface_solves_per_s": n[1] / sec,
            "sim_time_per_wall_s": {"min_member": st["t_min"] / sec, "max_member": st["t_max"] / sec}}


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["fp64_tflops"], "measured DFMA microbenchmark (profiles/fp64_peak.json)"
    return NOMINAL_FP64_TFLOPS, "nominal 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (no measurement)"


def ncu_traffic(workload_name):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(workload_name)
        if d:
            return d.get("bytes_per_launch")
    return None


def host_threads():
    """Host cores this process may use (the oracle's OpenMP thread count)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample_size(K, N, threads=1):
    return int(min(4096, max(1, round(1.5e8 * threads / (K * N)))))


def c5_cpu_cells(K, threads=1):
    """Oracle sample of C5: the first whole 4096-cell segments, ~6e7 cell-updates per host core
    (10-30 s of host-core time)."""
    return int(max(2, min(1024, round(6e7 * threads / (K * 4096))))) * 4096


def c4_cpu_members():
    """SURVEY §8(d)'s C4 subset: every 64th member plus the 32 with the largest single-phase
    star pressure of the converging vapour (all nucleating), in member order."""
    from oracle import oracle as O
    from paper_2211_00705_b200 import workloads as W
    w = W.c4(N=4)  # (the per-member data of C4 on a 4-cell stub: cells 0 and 3 carry rho, +u0 and -u0)
    M = w["M"]
    rho = w["rho"][:, 0]
    u0 = w["mom"][:, 0] / rho
    del w
    pstar = np.array([O.pressure(W.EOS_293K, O.VAP, O.single_phase_star(W.EOS_293K, O.VAP, rho[m], u0[m], rho[m], -u0[m]))
                      for m in range(M)])
    top = np.argsort(-pstar, kind="stable")[:32]
    return np.union1d(np.arange(0, M, 64), top)


def cpu_sample(name, K, threads):
    """(members or cells argument of workload(), description) of the oracle's bounded sample."""
    if name == "C5":
        S = c5_cpu_cells(max(K, 1), threads)
        return S, f"the first {S} cells (whole segments) of C5, {K} large steps from t=0"
    if name == "C4":
        mem = c4_cpu_members()
        return mem, (f"{len(mem)} members of C4 (every 64th + the 32 largest single-phase p*, SURVEY 8(d)), "
                     f"{K} large steps from t=0; throughput of the subset, extrapolated to the ensemble")
    if name in ("C1", "C2"):
        return None, f"{name}, {K} large steps from t=0"
    N = {"C3": 1024}[name]
    S = cpu_sample_size(max(K, 1), N, threads)
    return np.arange(S), f"members 0..{S - 1} of {name}, {K} large steps from t=0"


def run_oracle(name, members, steps, threads=1):
    from oracle import oracle as O
    w = workload(name, members)
    s = O.Sim(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"], threads=threads)
    s.set_state(w["rho"], w["mom"])
    t0 = time.perf_counter()
    st = s.step(steps) if "steps" in w else s.run_to(w["t_end"], steps)
    dt = time.perf_counter() - t0
    return st, dt


def cpu_baseline(name, K, warmup=0):
    """The oracle as it stands, OpenMP over the host's cores (members, or one grid's cells and
    regions), on a bounded sample of the workload."""
    th = host_threads()
    members, sample = cpu_sample(name, K, th)
    if warmup:
        run_oracle(name, 4096 if name == "C5" else (members[:th] if members is not None else None), warmup, th)
    st, dt = run_oracle(name, members, K, th)
    return {"value": st["cell_updates"] / dt, "unit": "cell-updates/s", "cores": th, "kind": "oracle",
            "sample": sample + f", {th} OpenMP threads"}, dt


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.workload
    cpu, dt = cpu_baseline(name, args.steps, args.warmup)
    v = cpu["value"]
    if name == "C5":
        cfg = {"workload": f"C5: one grid of {1 << 27} cells, 4096-cell random segments", "cells": 1 << 27,
               "parallelism": f"{cpu['cores']} host cores (CPU oracle, OpenMP)"}
    else:
        N = {"C3": 1024, "C4": 4096, "C1": 200, "C2": 1000}[name]
        cfg = {"workload": (f"{name}: {total_members(name)} members x {N} cells" +
                            (", cavitation ensemble" if name == "C3" else "")),
               "members": total_members(name), "cells_per_member": N,
               "parallelism": f"{cpu['cores']} host cores (CPU oracle, OpenMP)"}
    print(json.dumps({
        "impl": "reference", "metric": "fp64 cell-updates/s", "value": v, "unit": "cell-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the same workload as the eis arm's line; each step times a bounded sample of it
        "config": cfg, "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import torch.distributed as dist

    import paper_2211_00705_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.workload
    if name == "C5":
        return main_c5(args, torch, dist, P, world, rank, local)
    Mtot = args.members or total_members(name)
    # members interleaved over ranks (r, r + P, ...): the costly nucleating C4 members spread evenly
    # (SURVEY 8(e)); results do not depend on the sharding
    w = workload(name, np.arange(rank, Mtot, world) if name in ("C3", "C4") else None)
    stream = torch.cuda.current_stream()
    ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"], device=local,
                    stream=stream, threads=int(os.environ.get("EIS_THREADS", "0")),
                    tile_cells=int(os.environ.get("EIS_TILE", "0")), layout=int(os.environ.get("EIS_LAYOUT", "0")))
    rho_d = torch.from_numpy(w["rho"]).cuda()
    mom_d = torch.from_numpy(w["mom"]).cuda()
    t_end = w.get("t_end", float("inf"))

    def advance(k):
        if t_end == float("inf"):
            ctx.step(k)
        else:
            ctx.run_to(t_end, k)

    # warm-up (untimed), then reset to the initial state
    ctx.set_state(rho_d, mom_d)
    advance(args.warmup)
    torch.cuda.synchronize()
    ctx.set_state(rho_d, mom_d)
    cu0 = 0
    if args.start_steps:
        advance(args.start_steps)
        cu0 = ctx.step(0, stats=True)["cell_updates"]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.set_timing(True)  # CUDA events around the kernel on the library's (this) stream
    torch.cuda.synchronize()
    e0.record(stream)
    advance(args.steps)  # ONE launch of the member-resident kernel
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    kt = ctx.get_timing()
    ctx.set_timing(False)
    st = ctx.step(0, stats=True)  # counters of exactly the timed steps (set_state reset them)
    status = ctx.member_status()
    nbad = int((status != 0).sum())
    cu = st["cell_updates"] - cu0
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([cu, nbad], device="cuda", dtype=torch.int64)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        cu, nbad = int(c[0].item()), int(c[1].item())
    value = cu / (ms * 1e-3)
    rates = job_rates(dist, torch, world, st, ms)

    # end to end through the public API with pinned host buffers: set_state(host) + K steps
    # + get_state(host), one user call sequence per K steps
    e2e = None
    if not args.no_e2e:
        rho_h = torch.from_numpy(w["rho"]).pin_memory()
        mom_h = torch.from_numpy(w["mom"]).pin_memory()
        out = {"rho": torch.empty(w["rho"].shape, dtype=torch.float64).pin_memory(),
               "mom": torch.empty(w["rho"].shape, dtype=torch.float64).pin_memory(),
               "h": torch.empty(w["rho"].shape, dtype=torch.float64).pin_memory(),
               "n": torch.empty(w["M"], dtype=torch.int64).pin_memory(),
               "t": torch.empty(w["M"], dtype=torch.float64).pin_memory()}
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ctx.set_state(rho_h, mom_h)
        advance(args.steps)
        ctx.get_state(out)
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        cells = w["M"] * w["cap"] * world
        e2e = {"value": cu / te, "unit": "cell-updates/s",
               "h2d_bytes_per_step": 2 * 8 * cells / max(args.steps, 1),
               "d2h_bytes_per_step": (3 * 8 * cells + 16 * w["M"] * world) / max(args.steps, 1),
               "note": "one set_state(host pinned) + eis_step(K) + get_state(host pinned) sequence; bytes / K"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, _ = cpu_baseline(name, args.steps)

    cu_local = st["cell_updates"] - cu0 if world == 1 else None
    cu_gpu = cu / world if cu_local is None else cu_local
    try:
        ctx.tile_info()
        tiled = True  # AUTO layout: members with more than 2048 cells run on the tiled layout
    except P.EisError:
        tiled = False
    if tiled:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7700.0
        kms = kt["fast_ms"] if kt["fast_ms"] > 0 else ms
        achieved = C5_BYTES_PER_CELL_UPDATE * cu_gpu / (kms * 1e-3) / 1e9
        step_bw = C5_BYTES_PER_CELL_UPDATE * cu_gpu / (ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": ncu_traffic(name), "kernel": "eis::tiled_fast",
                "bytes_per_cell_update": C5_BYTES_PER_CELL_UPDATE,
                "kernel_ms_per_step": kms / max(args.steps, 1), "kernel_share_of_step": kms / ms,
                "window_ms_per_step": kt["window_ms"] / max(args.steps, 1),
                "tile_ms_per_step": kt["tile_ms"] / max(args.steps, 1),
                "whole_step_gbs": step_bw, "whole_step_frac": step_bw / hbm,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
        launches = kt["launches"]  # counted by the library (eis_get_timing)
        launch_note = ("per step: tiled_fast + window part A + dts_jobs + window part B + tiled_slow" +
                       (" + tiled_members_finish" if w["M"] > 1 else ""))
    else:
        peak, peak_src = fp64_peak()
        kms = kt["resident_ms"] if kt["resident_ms"] > 0 else ms
        achieved = FLOP_PER_CELL_UPDATE * cu_gpu / (kms * 1e-3) / 1e12  # per GPU
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": ncu_traffic(name), "kernel": "eis::resident_steps",
                "kernel_ms": kms, "kernel_share_of_step": kms / ms,
                "flop_per_cell_update": FLOP_PER_CELL_UPDATE, "peak_source": peak_src}
        launches = kt["launches"]
        launch_note = "one member-resident kernel launch for the K timed steps"
    if rank == 0:
        line = {
            "metric": "fp64 cell-updates/s", "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / max(args.steps, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64, BASELINE configs recipe)",
            "config": {"workload": f"{name}: {Mtot} members x {w['N']} cells, cavitation ensemble" if name == "C3"
                       else f"{name}: {Mtot} members x {w['N']} cells",
                       "members": Mtot, "cells_per_member": w["N"], "cell_capacity": w["cap"],
                       "parallelism": f"member-sharded dp{world} (interleaved)", "l2": "inputs (1.1 GB per GPU) larger than L2",
                       "layout": "tiled" if tiled else "member-resident", "launches": launch_note,
                       "implicit_regions": MODE_NAMES[w["params"].get("mode", 0)]},
            "roofline": roof,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "stats": {k: st[k] for k in ("cell_updates", "dts_iters", "iface_solves", "creations", "splits",
                                         "merges", "regions")},
            "members_not_ok": nbad, "rates": rates, "context": paper_context(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def paper_context():
    """The paper's speed-up of the split scheme over fully explicit local time stepping (north_star:
    quoted with its hardware -- unstated -- as context, not a target), and the same comparison
    measured on this GPU by tools/dts_vs_lts.py (profiles/r02_dts_vs_lts.json) when present."""
    ctx = {"paper_split_vs_explicit_lts": {
        "cavitation_E2": {"wall_time": 4.93 / 2.94, "local_iterations": 1941 / 355, "cite": "P:1324-1325"},
        "nucleation_E3": {"wall_time": 9811 / 509, "local_iterations": 27154016 / 1367460, "cite": "P:1435-1436"},
        "hardware": "unstated (1D CPU runs, ~400 cells)"}}
    f = os.path.join(ROOT, "profiles", "r02_dts_vs_lts.json")
    if os.path.exists(f):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            ctx["gpu_split_vs_explicit_lts"] = {
                "cavitation_E2": {"gpu_time": d["E2_ratio"]["gpu_time_lts_over_dts"],
                                  "local_iterations": d["E2_ratio"]["local_iterations_lts_over_dts"]},
                "nucleation_E3_first_7_steps": {"gpu_time": d["E3_ratio"]["gpu_time_lts_over_dts"],
                                                "local_iterations": d["E3_ratio"]["local_iterations_lts_over_dts"]},
                "source": "profiles/r02_dts_vs_lts.json (one B200)"}
        except (ValueError, KeyError):
            pass
    return ctx


def main_c5(args, torch, dist, P, world, rank, local):
    """BASELINE configs[4]: one 2^27-cell grid, tiled layout; world > 1 cuts it into rank slices."""
    from paper_2211_00705_b200 import workloads as W
    from paper_2211_00705_b200.decomp import RankGrid
    n_glob = args.members or (1 << 27)   # --members: profiling only, fewer cells
    w = with_mode(W.c5(n_cells=n_glob))
    stream = torch.cuda.current_stream()
    # world > 1: the per-step sequence (step_local, NCCL halo exchange + CFL all-reduce,
    # step_finish) replayed as CUDA graphs of EIS_RANK_GRAPH steps on the grid's own stream
    gsteps = int(os.environ.get("EIS_RANK_GRAPH", "10")) if world > 1 else 0
    rg = RankGrid(w["eos"], w["params"], w["N"], w["x_left"], w["x_right"], rank, world, device=local,
                  tile=int(os.environ.get("EIS_TILE", "1400")),
                  stream=stream, graph_steps=gsteps,
                  peer=os.environ.get("EIS_RANK_PEER", "1") != "0")  # the exchange over peer memory
    stream = rg.stream if rg.stream is not None else stream  # the library's stream: events go there
    rho_l = np.zeros(rg.cap)
    mom_l = np.zeros(rg.cap)
    rho_l[:rg.n] = w["rho"][0, rg.c0:rg.c1]
    mom_l[:rg.n] = w["mom"][0, rg.c0:rg.c1]
    mode = w["params"].get("mode", 0)
    del w
    rho_d = torch.from_numpy(rho_l).cuda()
    mom_d = torch.from_numpy(mom_l).cuda()
    rg.set_state(rho_d, mom_d)
    rg.step(args.warmup)
    torch.cuda.synchronize()
    rg.set_state(rho_d, mom_d)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rg.ctx.set_timing(gsteps == 0)  # CUDA events around each kernel on the library's (this) stream
    torch.cuda.synchronize()
    e0.record(stream)
    rg.step(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if gsteps:  # graph replays record no per-kernel events: the kernel times of the same steps, eager
        st_timed = rg.ctx.member_stats()[0]
        rg.set_state(rho_d, mom_d)
        torch.cuda.synchronize()
        rg.ctx.set_timing(True)
        rg.step(args.steps, graph=False)
        torch.cuda.synchronize()
    kt = rg.ctx.get_timing()
    rg.ctx.set_timing(False)
    st = rg.ctx.step(0, stats=True) if world == 1 else (st_timed if gsteps else rg.ctx.member_stats()[0])
    cu_local = st["cell_updates"]
    nbad = int(rg.ctx.member_status()[0] != 0)
    cu = st["cell_updates"]
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([cu, nbad, st["creations"]], device="cuda", dtype=torch.int64)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        cu, nbad = int(c[0].item()), int(c[1].item())
    value = cu / (ms * 1e-3)
    rates = job_rates(dist, torch, world, st, ms)

    e2e = None
    if not args.no_e2e:
        rho_h = torch.from_numpy(rho_l).pin_memory()
        mom_h = torch.from_numpy(mom_l).pin_memory()
        out = {k: torch.empty(rg.cap, dtype=torch.float64).pin_memory() for k in ("rho", "mom", "h")}
        out["n"] = torch.empty(1, dtype=torch.int64).pin_memory()
        out["t"] = torch.empty(1, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        rg.set_state(rho_h, mom_h)
        rg.step(args.steps)
        rg.ctx.get_state(out)
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        # a single grid moves only its live cells (rho, mom in; rho, mom, h, n, t out)
        e2e = {"value": cu / te, "unit": "cell-updates/s",
               "h2d_bytes_per_step": 2 * 8 * rg.n * world / max(args.steps, 1),
               "d2h_bytes_per_step": (3 * 8 * int(out["n"][0]) + 16) * world / max(args.steps, 1),
               "note": "one set_state(host pinned) + K steps + get_state(host pinned) per rank; bytes / K"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, _ = cpu_baseline("C5", args.steps)
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 7700.0
    # dominant kernel: the fast pass streams every cell of this rank's grid once per step
    achieved = C5_BYTES_PER_CELL_UPDATE * cu_local / (kt["fast_ms"] * 1e-3) / 1e9
    step_bw = C5_BYTES_PER_CELL_UPDATE * cu / (ms * 1e-3) / world / 1e9
    if rank == 0:
        line = {
            "metric": "fp64 cell-updates/s", "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / max(args.steps, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64, BASELINE configs[4] recipe)",
            "config": {"workload": f"C5: one grid of {n_glob} cells, 4096-cell random segments",
                       "cells": n_glob, "parallelism": f"tile-aligned grid slices x{world}, halo exchange + CFL min",
                       "l2": "state (2 GB) larger than L2",
                       "implicit_regions": MODE_NAMES[mode],
                       "launches": "per step: tiled_fast + window part A + dts_jobs + window part B + tiled_slow" +
                                   ("" if world == 1 else (" + tiled_finish (peer-memory exchange by the kernels)"
                                                           if rg.peer else " + NCCL halo exchange / all-reduce + tiled_finish"))
                                   + (f"; CUDA graphs of {gsteps} steps" if gsteps else "")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": ncu_traffic("C5"), "kernel": "eis::tiled_fast",
                         "bytes_per_cell_update": C5_BYTES_PER_CELL_UPDATE,
                         "kernel_ms_per_step": kt["fast_ms"] / max(args.steps, 1),
                         "kernel_share_of_step": kt["fast_ms"] / ms,
                         "window_ms_per_step": kt["window_ms"] / max(args.steps, 1),
                         "tile_ms_per_step": kt["tile_ms"] / max(args.steps, 1),
                         "whole_step_gbs": step_bw, "whole_step_frac": step_bw / hbm,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": kt["launches"], "clocks": clk,
            "stats": {k: st[k] for k in ("cell_updates", "dts_iters", "iface_solves", "creations", "splits",
                                         "merges", "regions")},
            "members_not_ok": nbad, "rates": rates, "context": paper_context(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
