#!/bin/bash
# Round-2 check b: GPU suite (incl. the Lax batches through the shared DTS loop), A/B of library variants
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b/pytest_gpu.log 2>&1; tail -12 gpurun_out/r2b/pytest_gpu.log
cp gpurun_out/decision_parity.json gpurun_out/r2b/ 2>/dev/null
for v in ${VARIANTS:-variants/*.so}; do
  for wl in C5 C4; do
    for st in 20 300; do
      [ $wl = C4 ] && [ $st = 300 ] && continue
      EIS_LIB=$PWD/$v timeout 600 python bench.py --workload $wl --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r2b/ab.json 2>gpurun_out/r2b/ab.err
      python -c "
import json
d=json.loads(open('gpurun_out/r2b/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl $st', 'value %.3e ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v, 4) for k, v in r.items() if k.endswith('ms_per_step') or k=='frac'})" 2>&1 | tail -1
    done
  done
done
