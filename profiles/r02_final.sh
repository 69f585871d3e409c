# r02 final refresh on the current code: GPU tests, bench lines for every config (+ reference
# arm on cfg2), the ncu launch list of the default bench command and full captures of the cfg2
# kernels (each ncu command runs only after the same command exited 0 without ncu).
O=gpurun_out/r02f
mkdir -p $O/bench
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest_gpu.log
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench/$c.json 2> $O/bench/$c.err; echo "$c rc=$?"
done
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench/reference_cfg2.json 2> $O/bench/reference_cfg2.err; echo "ref rc=$?"
for c in cfg1 cfg2 cfg3 cfg5; do
  timeout 600 python bench.py --config $c --levels 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench/${c}_depth0.json 2> /dev/null; echo "$c depth0 rc=$?"
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain.json 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo ncu1 rc=$?
python profiles/run_config.py cfg2 --iters 3 > /dev/null 2>&1; echo run_config rc=$?
ncu --set full --clock-control none --import-source on -k regex:modmm --launch-skip 2 -c 1 -f -o $O/modmm_cfg2 python profiles/run_config.py cfg2 --iters 3 > $O/ncu_modmm.log 2>&1; echo ncu2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:prep_tree --launch-skip 2 -c 1 -f -o $O/prep_tree_cfg2 python profiles/run_config.py cfg2 --iters 3 > $O/ncu_prep.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:post --launch-skip 4 -c 2 -f -o $O/post_cfg2 python profiles/run_config.py cfg2 --iters 3 > $O/ncu_post.log 2>&1; echo ncu4 rc=$?
python profiles/run_config.py cfg3 --iters 3 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:modmm --launch-skip 2 -c 1 -f -o $O/modmm_cfg3 python profiles/run_config.py cfg3 --iters 3 > $O/ncu_modmm3.log 2>&1; echo ncu5 rc=$?
