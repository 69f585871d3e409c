timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_multigpu.py -q -x 2>&1 | tail -1
for c in cfg2 cfg5 cfg3 cfg2 cfg5 cfg3; do
    echo "$c $(python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"], d["roofline"].get("phase_ms"))')"
done
