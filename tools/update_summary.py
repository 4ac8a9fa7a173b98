"""Refresh the bench rows of profiles/r01_summary.md from profiles/r01_bench_{c5,c4,c3}.json
(development tool; ncu rows are edited by hand)."""
import json, os, re
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
c5, c4, c3 = (json.load(open(os.path.join(P, f"r01_bench_{n}.json"))) for n in ("c5", "c4", "c3"))
r5, r4 = c5["roofline"], c4["roofline"]
rows = {
    "| C5 2^27 cells, 500 steps": f"| C5 2^27 cells, 500 steps (bench default) | fp64 cell-updates/s | {c5['value']:.3e} ({c5['ms_per_step']:.3f} ms/step); e2e {c5['e2e']['value']:.3e}; CPU oracle {c5['cpu_baseline']['value']:.3e} (1 core, 118,784-cell sample); clocks {c5['clocks']['sm_mhz']:.0f} MHz, reasons {c5['clocks']['reasons']} | r01_bench_c5.json |",
    "| C5 | roofline (hbm)": f"| C5 | roofline (hbm), dominant kernel `tiled_fast` | {r5['kernel_ms_per_step']:.3f} ms/step = {r5['achieved'] / 1e3:.2f} TB/s algorithmic (32 B/cell) = {100 * r5['frac']:.1f} % of 6544 GB/s; {100 * r5['kernel_share_of_step']:.0f} % of the step (ncu launch list of the same command: see below) | r01_bench_c5.json, r01_ncu_launches_c5_full.csv |",
    "| C5 | whole step": f"| C5 | whole step | {r5['whole_step_gbs'] / 1e3:.2f} TB/s at 32 B/cell = {100 * r5['whole_step_frac']:.0f} %; window full steps {r5['window_ms_per_step']:.3f} ms/step, whole tiles {r5['tile_ms_per_step']:.3f} ms/step | r01_bench_c5.json |",
    "| C4 16,384 x 4096, 2000 steps": f"| C4 16,384 x 4096, 2000 steps | fp64 cell-updates/s | {c4['value']:.3e} ({c4['ms_per_step']:.3f} ms/step, tiled layout through AUTO); e2e {c4['e2e']['value']:.3e}; CPU oracle {c4['cpu_baseline']['value']:.3e}; Newton mode (`--mode 3`, 300 steps) 9.96e10 vs DTS 8.49e10 | r01_bench_c4.json, r01_newton_vs_dts.json |",
    "| C4 | roofline (hbm)": f"| C4 | roofline (hbm), `tiled_fast` | {r4['kernel_ms_per_step']:.3f} ms/step = {r4['achieved'] / 1e3:.2f} TB/s = {100 * r4['frac']:.1f} %; window steps (2,395 one-cell droplets, ~30 DTS iterations each per step) {r4['window_ms_per_step']:.3f} ms/step | r01_bench_c4.json |",
    "| C3 65,536 x 1024, 2000 steps": f"| C3 65,536 x 1024, 2000 steps | fp64 cell-updates/s | {c3['value']:.3e} ({c3['ms_per_step']:.3f} ms/step); e2e {c3['e2e']['value']:.3e}; CPU oracle {c3['cpu_baseline']['value']:.3e} | r01_bench_c3.json |",
}
path = os.path.join(P, "r01_summary.md")
out = []
for line in open(path).read().split("\n"):
    for k, v in rows.items():
        if line.startswith(k):
            line = v
    out.append(line)
open(path, "w").write("\n".join(out))
print("\n".join(rows.values()))
