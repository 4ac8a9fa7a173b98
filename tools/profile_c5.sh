#!/bin/bash
# C5 round measurement: default bench line (K=500), ncu launch list of the same command (K=50),
# one full capture of each tiled kernel at step ~40 of the bench command.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -1 gpurun_out/bench_c5.json
python bench.py --steps 50 --no-cpu --no-e2e > gpurun_out/bench_c5_k50.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --steps 50 --no-cpu --no-e2e > gpurun_out/ncu_launches_c5.log 2>&1
for k in tiled_fast tiled_win tiled_slow; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
      -o gpurun_out/prof_bench_c5_$k python bench.py --steps 50 --no-cpu --no-e2e > gpurun_out/ncu_full_c5_$k.log 2>&1
done
ls -la gpurun_out | tail -5
python bench.py --workload C3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
bash tools/profile_c4.sh
ncu --set full --clock-control none --import-source on -k regex:resident_steps -s 1 -c 1 \
    -o gpurun_out/prof_bench_c3_resident python bench.py --workload C3 --steps 100 --no-cpu --no-e2e > gpurun_out/ncu_full_c3.log 2>&1
