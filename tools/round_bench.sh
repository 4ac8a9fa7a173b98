#!/bin/bash
# GPU suite, smoke, and the default bench lines (C5, C4, C3) with CPU baseline and e2e
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/rb
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/rb/gpu_tests.log 2>&1; tail -2 gpurun_out/rb/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for wl in C5 C4 C3; do
  timeout 900 python bench.py --workload $wl > gpurun_out/rb/bench_$wl.json 2> gpurun_out/rb/bench_$wl.err
  tail -1 gpurun_out/rb/bench_$wl.json | cut -c1-200
done
