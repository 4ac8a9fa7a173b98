#!/bin/bash
# Round measurement, ncu side (bench lines come from plain bench.py runs): launch list of the C5
# bench command (K=50), full captures of tiled_fast / tiled_win (C5, step ~40), tiled_fast (C4),
# resident_steps (C3); details exported as CSV on the box, only the C5 tiled_fast report kept.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/prof
O=gpurun_out/prof
python bench.py --steps 50 --no-cpu --no-e2e > $O/bench_c5_k50.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv \
    python bench.py --steps 50 --no-cpu --no-e2e > $O/ncu_launches_c5.log 2>&1
cap() {  # name kernel-regex skip bench-args...
  local name=$1 k=$2 s=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o $O/$name python bench.py "$@" \
      > $O/$name.log 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
}
cap c5_tiled_fast tiled_fast 40 --steps 50 --no-cpu --no-e2e
cap c5_tiled_win tiled_win 40 --steps 50 --no-cpu --no-e2e
cap c4_tiled_fast tiled_fast 40 --workload C4 --steps 50 --no-cpu --no-e2e
cap c3_resident resident_steps 1 --workload C3 --steps 100 --no-cpu --no-e2e
rm -f $O/c5_tiled_win.ncu-rep $O/c4_tiled_fast.ncu-rep $O/c3_resident.ncu-rep
du -sh $O
