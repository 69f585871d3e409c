timeout 600 python -m pytest tests/test_gpu_tree.py tests/test_gpu_combos.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do
for v in 1 0; do
  FSYRK_B200_POST2=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('post2=$v cfg2', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['post'])"
done
done
