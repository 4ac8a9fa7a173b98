#!/bin/bash
# window prediction: parity subset, then C5 / C4 with predictions on and off
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "${TESTS:-prediction or window or c5_tiled or tiled_ensemble or virtual_ranks_bitwise}" > gpurun_out/spec_tests.log 2>&1
tail -15 gpurun_out/spec_tests.log
for spec in ${SPECS:-1 0}; do
  for wl in ${WORKLOADS:-C5 C4}; do
    st=20; [ "$wl" = C4 ] && st=200
    EIS_WIN_SPEC=$spec EIS_WIN_EARLY_PER_SM=${EARLY:-8} timeout 900 python bench.py --workload $wl --steps $st --warmup 5 --no-cpu --no-e2e 2>gpurun_out/spec_${wl}_${spec}.err | tail -1 > gpurun_out/spec_${wl}_${spec}.json
    python - <<P
import json
try:
    d=json.load(open("gpurun_out/spec_${wl}_${spec}.json"))
    print("$wl spec=$spec value %.4e ms/step %.4f" % (d["value"], d["ms_per_step"]), {k:v for k,v in d["roofline"].items() if "ms" in k or k=="frac"}, d.get("kernel_ms_per_step"))
except Exception as ex:
    print("$wl spec=$spec failed", ex); print(open("gpurun_out/spec_${wl}_${spec}.err").read()[-1500:])
P
  done
done
