# ncu full capture of one kernel launch at a given C5 step: prof_c5_step.sh <kernel-regex> <launch-skip> <name>
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/$3 python tools/c5_variants.py recipe 8 > gpurun_out/$3.log 2>&1
tail -1 gpurun_out/$3.log
