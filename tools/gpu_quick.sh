#!/bin/bash
# GPU check: the -m gpu suite, then the C5 and C4 bench lines without CPU baseline / e2e
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/q_c5.json 2> gpurun_out/q_c5.err; tail -1 gpurun_out/q_c5.json | cut -c1-420
timeout 300 python bench.py --workload C4 --no-cpu --no-e2e > gpurun_out/q_c4.json 2> gpurun_out/q_c4.err; tail -1 gpurun_out/q_c4.json | cut -c1-420
python - <<'P'
import json
for f in ("gpurun_out/q_c5.json", "gpurun_out/q_c4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f, "value %.3e ms/step %.3f fast %.3f win %.3f tile %.3f frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms_per_step"], r["window_ms_per_step"], r["tile_ms_per_step"], r["frac"]), d["stats"])
    except Exception as ex:
        print(f, "failed", ex)
P
