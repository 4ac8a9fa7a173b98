#!/bin/bash
# C4 knob sweep (dev): tile size and early part-A CTAs per SM with window prediction
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
run() { name=$1; shift
  env "$@" timeout 300 python bench.py --workload C4 --no-cpu --no-e2e > gpurun_out/sw_$name.json 2> gpurun_out/sw_$name.err
  python - <<P
import json
try:
    d=json.loads(open("gpurun_out/sw_$name.json").read().strip().splitlines()[-1])
    print("$name", "%.4e" % d["value"], "%.4f ms" % d["ms_per_step"], d["members_not_ok"], {k:round(v,4) for k,v in d["roofline"].items() if "ms" in k})
except Exception as ex: print("$name no json", ex); print(open("gpurun_out/sw_$name.err").read()[-300:])
P
}
run t1400 EIS_TILE=1400
run t1366 EIS_TILE=1366
run t2048 EIS_TILE=2048
run t1024 EIS_TILE=1024
run t4096 EIS_TILE=4096
run e4 EIS_WIN_EARLY_PER_SM=4
run e12 EIS_WIN_EARLY_PER_SM=12
