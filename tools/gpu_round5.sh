#!/bin/bash
# session-5 evidence: full GPU suite, smoke, the bench lines (C5 driver's command, C5 500 steps, C4, C3),
# then (each after its command exited 0 without ncu) the ncu launch lists of the C5 and C4 commands
# and one --set full capture of a steady-state tiled_fast launch of the C5 command
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r5_tests.log 2>&1; tail -3 gpurun_out/r5_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
run() { name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/r5_$name.json 2> gpurun_out/r5_$name.err
  echo "$name rc=$?"
  python - <<P
import json
try:
    d=json.loads(open("gpurun_out/r5_$name.json").read().strip().splitlines()[-1])
    print("  ", "%.4e" % d["value"], "%.4f ms" % d["ms_per_step"], d["members_not_ok"], "frac %.4f" % d["roofline"]["frac"], {k:round(v,4) for k,v in d["roofline"].items() if "ms" in k}, "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "launches", d.get("gpu_launches"))
except Exception as ex: print("  no json", ex); print(open("gpurun_out/r5_$name.err").read()[-600:])
P
}
run c5 --steps 20 --warmup 5
run c5_500 --no-cpu --no-e2e
run c4 --workload C4
run c3 --workload C3 --no-cpu
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r5_ncu_launches_c4.csv python bench.py --workload C4 --steps 60 --warmup 3 --no-cpu --no-e2e > gpurun_out/r5_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r5_ncu_launches_c5.csv python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r5_ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled_fast -s 15 -c 1 -o gpurun_out/r5_ncu_full_tiled_fast python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r5_ncu_full.log 2>&1; echo "ncu full rc=$?"; ls -la gpurun_out/r5_ncu_full_tiled_fast.ncu-rep
