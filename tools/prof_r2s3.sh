#!/bin/bash
# Round-2 source-level captures: tiled_fast (steady state) and dts_jobs (creation transient) of the
# driver's C5 command (20 steps from t=0), --set full with source counters.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/p3; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tiled_fast" -s 6 -c 1 -o $O/fast python bench.py --steps 8 --warmup 0 --no-cpu --no-e2e > $O/ncu_fast.log 2>&1; tail -2 $O/ncu_fast.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dts_jobs" -s 1 -c 2 -o $O/dts python bench.py --steps 4 --warmup 0 --no-cpu --no-e2e > $O/ncu_dts.log 2>&1; tail -2 $O/ncu_dts.log
ls -la $O
