#!/bin/bash
# quick A/B of variants/*.so on C5 (driver command: 20 steps from t=0)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
STEPS=${STEPS:-20} WORKLOADS=${WORKLOADS:-C5} bash tools/ab_libs.sh
