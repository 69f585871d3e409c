timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "131071 or golden or extreme or accumulator" 2>&1 | tail -1
FSYRK_B200_LIB=profiles/variants/ktrace.so python profiles/ktrace.py cfg2 2>&1 | grep -A6 "^tile" | head -6
for c in cfg2 cfg5 cfg2 cfg5; do
    echo "$c $(python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"], d["roofline"]["frac"], d["roofline"].get("phase_ms"))')"
done
