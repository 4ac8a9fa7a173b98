#!/bin/bash
# parity subset of the tiled paths and the C5 A/B for each variant in $VARIANTS
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in $VARIANTS; do
  EIS_LIB=$PWD/$v timeout 600 python -m pytest tests -m gpu -x -q -k "c5_tiled or c5_virtual or window_path or c4_members or tiled_ensemble or ragged" > gpurun_out/vc_$(basename $v).log 2>&1; echo "$v tests: $(tail -1 gpurun_out/vc_$(basename $v).log)"
done
STEPS=${STEPS:-20} WORKLOADS=${WORKLOADS:-C5} bash tools/ab_libs.sh
