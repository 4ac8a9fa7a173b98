#!/bin/bash
# A/B of library variants on C3 (300 steps), C5 (20), C4 (20); then the GPU suite on the in-tree build
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/ab3
for v in ${VARIANTS:-variants/*.so}; do
  for cfg in "C3 300" "C5 20" "C4 20"; do
    set -- $cfg
    EIS_LIB=$PWD/$v timeout 600 python bench.py --workload $1 --steps $2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab3/ab.json 2>gpurun_out/ab3/ab.err
    python -c "
import json
d=json.loads(open('gpurun_out/ab3/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $1 $2', 'value %.3e ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v, 4) for k, v in r.items() if k.endswith('ms_per_step') or k=='frac'})" 2>&1 | tail -1
  done
done
[ -n "$NOTEST" ] || { timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab3/pytest_gpu.log 2>&1; tail -4 gpurun_out/ab3/pytest_gpu.log; }
