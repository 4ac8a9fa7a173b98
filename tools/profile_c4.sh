#!/bin/bash
# C4 (16384 x 4096 ensemble, AUTO -> tiled layout): default bench line, ncu launch list (K=50),
# one full capture of tiled_fast at step ~40 of the same command.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python bench.py --workload C4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -1 gpurun_out/bench_c4.json
python bench.py --workload C4 --steps 50 --no-cpu --no-e2e > gpurun_out/bench_c4_k50.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --workload C4 --steps 50 --no-cpu --no-e2e > gpurun_out/ncu_launches_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tiled_fast -s 40 -c 1 \
    -o gpurun_out/prof_bench_c4_tiled_fast python bench.py --workload C4 --steps 50 --no-cpu --no-e2e \
    > gpurun_out/ncu_full_c4.log 2>&1
ls -la gpurun_out | tail -5
