# r02 refresh on the current code: bench lines for every config (+ reference arm), then the ncu
# launch list of the default bench command and full captures of the cfg2 kernels (each ncu
# command runs only after the same command exited 0 without ncu).
mkdir -p gpurun_out/r02/bench
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02/bench/$c.json 2> gpurun_out/r02/bench/$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02/bench/reference_cfg2.json 2> gpurun_out/r02/bench/reference_cfg2.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02/plain.json 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/ncu_launch.log 2>&1; echo ncu1 rc=$?
python profiles/run_config.py cfg2 --iters 3 > /dev/null 2>&1; echo run_config rc=$?
ncu --set full --clock-control none --import-source on -k regex:modmm --launch-skip 2 -c 1 -f -o gpurun_out/r02/modmm_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/r02/ncu_modmm.log 2>&1; echo ncu2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:prep_tree --launch-skip 2 -c 1 -f -o gpurun_out/r02/prep_tree_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/r02/ncu_prep.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:post --launch-skip 6 -c 3 -f -o gpurun_out/r02/post_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/r02/ncu_post.log 2>&1; echo ncu4 rc=$?
