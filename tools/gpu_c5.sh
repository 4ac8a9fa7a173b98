cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/c5_variants.py uniform 60 2>&1 | cut -c1-200
PERSTEP=1 timeout 300 python tools/c5_variants.py recipe 60 2>&1 | cut -c1-900
timeout 300 python bench.py --steps 500 --no-cpu --no-e2e | cut -c1-250
