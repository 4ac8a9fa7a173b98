#!/bin/bash
# C3 (member-resident) A/B of $VARIANTS: value and ms/step
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in $VARIANTS; do
  EIS_LIB=$PWD/$v timeout 600 python bench.py --workload C3 --steps ${STEPS:-300} --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v C3', 'value %.4e ms/step %.4f frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['frac']))"
done
