#!/bin/bash
# Round-2 evidence: driver-style bench lines (C5 default, C4, C3), the reference arm, smoke, the
# ncu launch list of the C5 bench command and one ncu --set full capture of each C5 step kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/p2; mkdir -p $O
nproc > $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref_c5.json 2> $O/ref_c5.err; tail -1 $O/ref_c5.json | cut -c1-250
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c5.json 2> $O/bench_c5.err; tail -1 $O/bench_c5.json | cut -c1-250
timeout 900 python bench.py --workload C4 > $O/bench_c4.json 2> $O/bench_c4.err; tail -1 $O/bench_c4.json | cut -c1-200
timeout 900 python bench.py --workload C3 > $O/bench_c3.json 2> $O/bench_c3.err; tail -1 $O/bench_c3.json | cut -c1-200
timeout 900 python bench.py --steps 500 --no-cpu --no-e2e > $O/bench_c5_500.json 2> $O/bench_c5_500.err; tail -1 $O/bench_c5_500.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/ncu_ll.log 2>&1; tail -1 $O/ncu_ll.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"tiled_fast|tiled_win|dts_jobs" -s 20 -c 4 -o $O/c5_kernels python bench.py --steps 8 --warmup 0 --no-cpu --no-e2e > $O/ncu_full.log 2>&1; tail -1 $O/ncu_full.log
