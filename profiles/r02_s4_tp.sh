timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_configs.py tests/test_gpu_combos.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do
for c in cfg2; do
python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', d['ms_per_step'], d['parity'], r['phase_ms'], r['frac'], {k:(v['frac'] if isinstance(v,dict) else v) for k,v in r['elementwise_hbm'].items() if k in ('pre','post','convert')})"
done
done
python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg4', d['ms_per_step'], d['parity'], r['phase_ms'], r['frac'], {k:(v['frac'] if isinstance(v,dict) else v) for k,v in r['elementwise_hbm'].items() if k in ('pre','post','convert')})"
