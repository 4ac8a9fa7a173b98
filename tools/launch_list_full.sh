#!/bin/bash
# ncu launch list of the full default C5 bench command (500 timed steps; kernel shares comparable
# with the bench line's), then the default bench lines (C5, C4, C3)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/ll
for wl in C5 C4 C3; do
  timeout 900 python bench.py --workload $wl > gpurun_out/ll/bench_$wl.json 2> gpurun_out/ll/bench_$wl.err
  tail -1 gpurun_out/ll/bench_$wl.json | cut -c1-150
done
python bench.py --no-cpu --no-e2e > gpurun_out/ll/bench_c5_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/ll/launches_c5_full.csv \
    python bench.py --no-cpu --no-e2e > gpurun_out/ll/ncu_launches_c5_full.log 2>&1
tail -2 gpurun_out/ll/ncu_launches_c5_full.log
