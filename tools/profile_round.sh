#!/bin/bash
# Round measurement: default bench line, ncu launch list of the same command, one full
# capture of the dominant kernel (resident_steps, bench config with K=100 steps).
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -1 gpurun_out/bench_default.json
python bench.py --steps 100 --no-cpu --no-e2e > gpurun_out/bench_k100.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 100 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:resident_steps -s 1 -c 1 \
    -o gpurun_out/prof_bench python bench.py --steps 100 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
python bench.py --workload C4 --members 2048 --steps 200 --no-cpu --no-e2e > gpurun_out/bench_c4_sample.json 2>&1
python tools/c5_full.py 100 > gpurun_out/c5_full.log 2>&1
