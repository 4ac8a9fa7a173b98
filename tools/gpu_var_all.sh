#!/bin/bash
# numerics variants: the whole GPU suite per variant, then C5 / C4 / C3 A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in $VARIANTS; do
  EIS_LIB=$PWD/$v timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/va_$(basename $v).log 2>&1; echo "$v tests: $(tail -1 gpurun_out/va_$(basename $v).log)"
  grep -E "^FAILED" gpurun_out/va_$(basename $v).log | head -5
done
STEPS=20 WORKLOADS="C5 C4" bash tools/ab_libs.sh
STEPS=300 bash tools/ab_c3.sh
