set -x
timeout 600 python tools/parity_probe.py 2>&1 | tee gpurun_out/probe2.log
for mb in 4 3 2; do EIS_RESIDENT_MINB=$mb timeout 600 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | tee gpurun_out/bench_v2_minb$mb.log; done
