#!/bin/bash
# session-5 evidence: full GPU suite, then C5 (driver's command and 500 steps) with predictions off / on, C4, C3
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r5_tests.log 2>&1; tail -3 gpurun_out/r5_tests.log
run() { # name, args..., env via ENVV
  name=$1; shift
  env $ENVV timeout 900 python bench.py "$@" > gpurun_out/r5_$name.json 2> gpurun_out/r5_$name.err
  echo "$name rc=$?"
  python - <<P
import json
try:
    d=json.loads(open("gpurun_out/r5_$name.json").read().strip().splitlines()[-1])
    print("  ", "%.4e" % d["value"], "%.4f ms" % d["ms_per_step"], d["members_not_ok"], "frac %.4f" % d["roofline"]["frac"], {k:round(v,4) for k,v in d["roofline"].items() if "ms" in k}, "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
except Exception as ex: print("  no json", ex); print(open("gpurun_out/r5_$name.err").read()[-600:])
P
}
ENVV="EIS_WIN_SPEC=0" run c5_500_spec0 --workload C5 --steps 500 --no-cpu --no-e2e
ENVV="EIS_WIN_SPEC=1" run c5_500_spec1 --workload C5 --steps 500 --no-cpu --no-e2e
ENVV="EIS_WIN_SPEC=1" run c5_20_spec1 --workload C5 --steps 20 --warmup 5 --no-cpu --no-e2e
ENVV="EIS_WIN_SPEC=0" run c4_spec0 --workload C4 --no-cpu --no-e2e
ENVV="X=1" run c4 --workload C4
ENVV="X=1" run c5 --steps 20 --warmup 5
