timeout 600 python -m pytest tests/test_gpu_tree.py tests/test_gpu_combos.py tests/test_gpu_lowmem.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for v in "FSYRK_B200_POST2=1" "FSYRK_B200_POST2=0" "FSYRK_B200_LIB=build_variants/lib_post32.so"; do
  env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg2', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['post'])"
  env $v python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg4', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['post'])"
done
done
