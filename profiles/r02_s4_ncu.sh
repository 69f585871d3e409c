# session-4 ncu captures of the cfg2 elementwise kernels (source-level), after a clean plain run
mkdir -p gpurun_out/s4
python profiles/run_config.py cfg2 --iters 3 > gpurun_out/s4/plain.log 2>&1; echo plain rc=$?
ncu --set full --clock-control none --import-source on -k regex:prep_tree --launch-skip 2 -c 1 -f -o gpurun_out/s4/prep_tree_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/s4/ncu_prep.log 2>&1; echo ncu prep rc=$?
ncu --set full --clock-control none --import-source on -k regex:post --launch-skip 4 -c 2 -f -o gpurun_out/s4/post_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/s4/ncu_post.log 2>&1; echo ncu post rc=$?
