#!/bin/bash
# the whole GPU suite on the in-tree build, then the C5 / C4 A/B of $VARIANTS
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/full_tests.log)"
grep -E "FAIL|Error|assert" gpurun_out/full_tests.log | head -10
STEPS=${STEPS:-20} WORKLOADS=${WORKLOADS:-C5 C4} bash tools/ab_libs.sh
