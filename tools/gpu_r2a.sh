#!/bin/bash
# Round-2 check: GPU suite, A/B of HEAD vs working-tree library in the driver's bench config,
# then one ncu capture of the window kernel in that config.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/r2a
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2a/pytest_gpu.log 2>&1; tail -8 gpurun_out/r2a/pytest_gpu.log
cp gpurun_out/decision_parity.json gpurun_out/r2a/ 2>/dev/null
for v in variants/a_head.so variants/b_work.so; do
  for wl in C5 C4 C3; do
    for st in 20 300; do
      [ $wl = C3 ] && [ $st = 300 ] && continue
      EIS_LIB=$PWD/$v timeout 600 python bench.py --workload $wl --steps $st --warmup 5 --no-cpu --no-e2e > gpurun_out/r2a/ab.json 2>gpurun_out/r2a/ab.err
      python -c "
import json
d=json.loads(open('gpurun_out/r2a/ab.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $wl $st', 'value %.3e ms/step %.3f' % (d['value'], d['ms_per_step']), {k: round(v, 4) for k, v in r.items() if k.endswith('ms_per_step') or k=='frac'})" 2>&1 | tail -1
    done
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled_win -s 4 -c 1 -o gpurun_out/r2a/win_c5 python bench.py --steps 8 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2a/ncu_win.log 2>&1; tail -3 gpurun_out/r2a/ncu_win.log
