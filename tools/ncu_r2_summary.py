"""Summaries for profiles/ (dev tool): per-kernel key metrics of an ncu --set full report and the
per-kernel share of a launch list (ncu --metrics gpu__time_duration.sum --csv).
usage: python tools/ncu_r2_summary.py report.ncu-rep launches.csv > summary.txt"""
import collections, csv, io, subprocess, sys

KEYS = [("gpu__time_duration.sum", "duration"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
        ("sm__inst_executed.avg.per_cycle_active", "IPC"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("launch__registers_per_thread", "registers/thread"),
        ("smsp__average_warp_latency_per_inst_issued.ratio", "cycles per issued inst (warp)"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long scoreboard"),
        ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall no instruction"),
        ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per inst")]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = rows[1]
    for r in rows[2:]:
        print(f"== {r[h.index('Kernel Name')][:90]}")
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                print(f"   {name:32s} {r[i]} {units[i]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}
    agg = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > iV:
            agg[r[iN].split("(")[0]].append(float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0))
    step = [k for k in agg if any(s in k for s in ("tiled_fast", "tiled_win", "dts_jobs", "tiled_slow"))]
    tot = sum(sum(agg[k]) for k in step)
    print("== launch list (ncu, serialised, cold caches): step kernels")
    for k in step:
        v = agg[k]
        print(f"   {k[:60]:60s} n={len(v):4d} mean {sum(v) / len(v):9.1f} us  share of step kernels {100 * sum(v) / tot:5.1f} %")


if __name__ == "__main__":
    full(sys.argv[1])
    if len(sys.argv) > 2:
        launches(sys.argv[2])
