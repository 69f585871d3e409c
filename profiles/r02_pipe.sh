FSYRK_B200_POST_PIPE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_combos.py tests/test_gpu_lowmem.py tests/test_multigpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for v in 1 0; do
 for c in "cfg2 --steps 10" "cfg3 --steps 10" "cfg5 --steps 5"; do
  FSYRK_B200_POST_PIPE=$v python bench.py --config $c --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pipe=$v', '$c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['post'])"
 done
done
done
