mkdir -p gpurun_out/r02
timeout 300 python -m pytest tests/test_gpu_tree.py -x -q > gpurun_out/r02/tree_tests.log 2>&1; echo tree tests rc=$?; tail -2 gpurun_out/r02/tree_tests.log
for t in 1 0; do
  FSYRK_B200_TREE_PREP=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/bench_tree$t.json 2>gpurun_out/r02/bench_tree$t.err; echo bench tree=$t rc=$?
  python -c "
import json; d=json.load(open('gpurun_out/r02/bench_tree$t.json'))
print('tree=$t', d['ms_per_step'], d['value'], d['parity'], d['roofline']['phase_ms'], d['roofline']['elementwise_hbm']['pre'])"
done
./profiles/ubench/ubench_dmma > gpurun_out/r02/ubench_dmma.txt 2>&1; cat gpurun_out/r02/ubench_dmma.txt
python profiles/run_config.py cfg2 --iters 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:prep_tree --launch-skip 1 -c 1 -f -o gpurun_out/r02/prep_tree_cfg2 python profiles/run_config.py cfg2 --iters 3 > gpurun_out/r02/ncu_tree.log 2>&1; echo ncu rc=$?
