#!/bin/bash
# Round-2 check e: the window split. Its parity tests first, then A/B (split on/off), then the suite.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "split or k5 or window_path or c5_tiled_against or full_size_block" > gpurun_out/r2e/pytest_split.log 2>&1; tail -4 gpurun_out/r2e/pytest_split.log
for sp in 1 0; do
  for wl in C5 C4; do
    for st in 20 300; do
      [ $wl != C5 ] && [ $st = 300 ] && continue
      EIS_WIN_SPLIT=$sp timeout 600 python bench.py --workload $wl --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r2e/ab.json 2>gpurun_out/r2e/ab.err
      python -c "
import json
d=json.loads(open('gpurun_out/r2e/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('split=$sp $wl $st', 'value %.3e ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v, 4) for k, v in r.items() if k.endswith('ms_per_step') or k=='frac'}, d['stats']['dts_iters'])" 2>&1 | tail -1
    done
  done
done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2e/pytest_gpu.log 2>&1; tail -4 gpurun_out/r2e/pytest_gpu.log
