cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
WL=C4 timeout 300 python tools/window_diag.py 1 50 500 1500 2>&1 | tail -12
WL=C4 EIS_LIB=$PWD/variants/phase.so timeout 300 python tools/window_phases.py 50 1000 2>&1 | tail -16
for pol in 1 2 4; do EIS_WIN_POLL_PER_SM=$pol VARIANTS=paper_2211_00705_b200/libeis.so WORKLOADS=C4 bash tools/ab_libs.sh; done
