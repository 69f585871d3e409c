# r01 profile set for cfg2: launch list of the bench command, then full ncu captures of one
# launch of each hot kernel (each command first ran cleanly without ncu in profiles/full_bench.sh)
set -x
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:modmm --launch-skip 2 -c 1 -f -o gpurun_out/modmm_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/ncu_modmm.log 2>&1; echo ncu2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:prep_vec --launch-skip 6 -c 3 -f -o gpurun_out/prep_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/ncu_prep.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:post --launch-skip 6 -c 3 -f -o gpurun_out/post_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/ncu_post.log 2>&1; echo ncu4 rc=$?
ncu --set full --clock-control none -k regex:modmm --launch-skip 1 -c 1 -f -o gpurun_out/modmm_cfg5 python profiles/run_config.py cfg5 --iters 2 > gpurun_out/ncu_modmm5.log 2>&1; echo ncu5 rc=$?
