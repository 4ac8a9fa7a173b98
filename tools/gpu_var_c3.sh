#!/bin/bash
# resident-kernel variants: parity subset (C1-C4 resident paths, windows) and the C3 / C5 A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in $VARIANTS; do
  EIS_LIB=$PWD/$v timeout 900 python -m pytest tests -m gpu -x -q -k "c1 or c2 or c3 or c4_members or 363K or decision or lts_mode_c2 or window or c5_tiled" > gpurun_out/vr_$(basename $v).log 2>&1; echo "$v tests: $(tail -1 gpurun_out/vr_$(basename $v).log)"
done
STEPS=${STEPS:-300} WORKLOADS="C3" bash tools/ab_libs.sh 2>&1 | sed 's/fast.*//'
STEPS=20 WORKLOADS="C5" bash tools/ab_libs.sh
