cd $GRAFT_REPO_ROOT
for v in uniform calm recipe; do timeout 300 python tools/c5_variants.py $v 60; done > gpurun_out/c5_variants.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tiled_step -s 40 -c 1 -o gpurun_out/prof_c5_recipe python tools/c5_variants.py recipe 50 > gpurun_out/ncu_c5_recipe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tiled_step -s 40 -c 1 -o gpurun_out/prof_c5_uniform python tools/c5_variants.py uniform 50 > gpurun_out/ncu_c5_uniform.log 2>&1
cat gpurun_out/c5_variants.log
