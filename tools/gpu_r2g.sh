#!/bin/bash
# Profile of the split window path in the driver's bench configuration (C5, 20 steps from t=0)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2g
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g/bench.json 2> gpurun_out/r2g/bench.err; tail -1 gpurun_out/r2g/bench.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2g/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2g/ncu_ll.log 2>&1; tail -2 gpurun_out/r2g/ncu_ll.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"dts_jobs|tiled_win" -s 12 -c 3 -o gpurun_out/r2g/split_c5 python bench.py --steps 8 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2g/ncu_full.log 2>&1; tail -2 gpurun_out/r2g/ncu_full.log
