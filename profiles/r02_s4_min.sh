# branch-free mod add/sub/mulc (VIADDMNMX) + lazy phase events: full GPU tests, then every config
mkdir -p gpurun_out/s4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4/pytest_gpu_min.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s4/pytest_gpu_min.log
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', d['ms_per_step'], d['parity'], r['phase_ms'], r['frac'], {k:(v['frac'] if isinstance(v,dict) else v) for k,v in r['elementwise_hbm'].items() if k in ('pre','post','convert')})"
done
