#!/bin/bash
# quick check: split parity tests, then the C5 (20, 300 steps) and C4 bench lines
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/q2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "${TESTK:-split or k5 or window_path or full_size_block}" > gpurun_out/q2/pytest.log 2>&1; tail -3 gpurun_out/q2/pytest.log
for wl in C5 C4; do
  for st in 20 300; do
    [ $wl != C5 ] && [ $st = 300 ] && continue
    timeout 600 python bench.py --workload $wl --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/q2/ab.json 2>gpurun_out/q2/ab.err
    python -c "
import json
d=json.loads(open('gpurun_out/q2/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$wl $st', 'value %.3e ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v, 4) for k, v in r.items() if k.endswith('ms_per_step') or k=='frac'})" 2>&1 | tail -1
  done
done
