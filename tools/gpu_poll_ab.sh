#!/bin/bash
# part A of the window step polling beside tiled_fast (EIS_WIN_POLL_PER_SM): parity and C5 / C4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for k in ${POLLS:-0 1 2}; do
  if [ "$k" != "0" ]; then
    EIS_WIN_POLL_PER_SM=$k timeout 900 python -m pytest tests -m gpu -x -q -k "c5_tiled or window or c4_members or tiled_ensemble or full_size or virtual" > gpurun_out/poll_$k.log 2>&1; echo "poll $k tests: $(tail -1 gpurun_out/poll_$k.log)"
  fi
  for wl in C5 C4; do
    EIS_WIN_POLL_PER_SM=$k timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('poll $k $wl', 'value %.4e ms/step %.4f fast %.4f win %.4f' % (d['value'], d['ms_per_step'], r['kernel_ms_per_step'], r['window_ms_per_step']))"
  done
done
