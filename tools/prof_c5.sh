# ncu full capture of one tiled kernel launch on a C5 variant: prof_c5.sh <variant> <kernel-regex> <name>
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 40 -c 1 -o gpurun_out/$3 python tools/c5_variants.py $1 50 > gpurun_out/$3.log 2>&1
tail -1 gpurun_out/$3.log
