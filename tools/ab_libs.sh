#!/bin/bash
# A/B of library builds (development tool): bench lines of C5 and C4 for each variants/*.so
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in ${VARIANTS:-variants/*.so}; do
  for wl in ${WORKLOADS:-C5 C4}; do
    EIS_LIB=$PWD/$v timeout 300 python bench.py --workload $wl --steps ${STEPS:-300} --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
    python -c "
import json,sys
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl', 'value %.3e ms/step %.3f fast %.3f win %.3f tile %.3f' % (d['value'], d['ms_per_step'], r['kernel_ms_per_step'], r['window_ms_per_step'], r['tile_ms_per_step']))" 2>&1 | tail -1
  done
done
