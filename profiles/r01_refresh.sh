# r01 refresh on the current code: GPU tests, bench lines for every config (+ reference arm),
# then the ncu launch list of the default bench command and full captures of the hot kernels
# (each ncu command runs only after the same command exited 0 without ncu).
mkdir -p gpurun_out/r01 gpurun_out/r01/bench
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/r01/pytest_gpu.log
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r01/bench/$c.json 2> gpurun_out/r01/bench/$c.err; echo "$c rc=$?"
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01/bench/reference_cfg2.json 2> gpurun_out/r01/bench/reference_cfg2.err; echo "ref rc=$?"
python bench.py > gpurun_out/r01/bench/default.json 2> gpurun_out/r01/bench/default.err; echo "default rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01/plain.json 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01/ncu_launch.log 2>&1; echo ncu1 rc=$?
python profiles/run_config.py cfg2 --iters 3 > /dev/null 2>&1; echo run_config rc=$?
ncu --set full --clock-control none --import-source on -k regex:modmm --launch-skip 2 -c 1 -f -o gpurun_out/r01/modmm_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/r01/ncu_modmm.log 2>&1; echo ncu2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:prep_vec --launch-skip 6 -c 3 -f -o gpurun_out/r01/prep_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/r01/ncu_prep.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:post --launch-skip 6 -c 3 -f -o gpurun_out/r01/post_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/r01/ncu_post.log 2>&1; echo ncu4 rc=$?
python profiles/run_config.py cfg5 --iters 2 > /dev/null 2>&1; echo run_config5 rc=$?
ncu --set full --clock-control none -k regex:modmm --launch-skip 1 -c 1 -f -o gpurun_out/r01/modmm_cfg5 python profiles/run_config.py cfg5 --iters 2 > gpurun_out/r01/ncu_modmm5.log 2>&1; echo ncu5 rc=$?
python profiles/run_config.py cfg3 --iters 2 > /dev/null 2>&1; echo run_config3 rc=$?
ncu --set full --clock-control none -k regex:modmm --launch-skip 1 -c 1 -f -o gpurun_out/r01/modmm_cfg3 python profiles/run_config.py cfg3 --iters 2 > gpurun_out/r01/ncu_modmm3.log 2>&1; echo ncu6 rc=$?
python profiles/run_config.py cfg4 --iters 2 > /dev/null 2>&1; echo run_config4 rc=$?
ncu --set full --clock-control none -k regex:modmm --launch-skip 1 -c 1 -f -o gpurun_out/r01/modmm_cfg4 python profiles/run_config.py cfg4 --iters 2 > gpurun_out/r01/ncu_modmm4.log 2>&1; echo ncu7 rc=$?
