# fused two-level post: step loop rolled (shipped candidate) vs fully unrolled
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_configs.py tests/test_gpu_combos.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_post2_unroll.so; do
for c in "cfg2 --steps 20" "cfg4 --steps 4"; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config $c --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $c', d['ms_per_step'], d['parity'], r['phase_ms']['post'], r['elementwise_hbm']['post']['frac'])"
done
done
done
