#!/bin/bash
# DTS (mode 0) vs Newton (mode 3) on the bench workloads (short runs, no CPU baseline / e2e)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for wl in C4 C5 C3; do
  for m in 0 3; do
    timeout 300 python bench.py --workload $wl --mode $m --steps ${STEPS:-300} --no-cpu --no-e2e > gpurun_out/nb.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/nb.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$wl mode $m', 'value %.3e ms/step %.3f' % (d['value'], d['ms_per_step']), 'win %.3f' % r.get('window_ms_per_step', -1), 'dts_iters', d['stats']['dts_iters'], 'regions', d['stats']['regions'], 'bad', d['members_not_ok'])"
  done
done
