run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 lib=$(basename ${FSYRK_B200_LIB:-default})', d['ms_per_step'], d['roofline']['phase_ms'], d['parity'])"; }
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in cfg2 cfg3 cfg5 cfg4; do run $c; FSYRK_B200_LIB=$PWD/profiles/variants/nostagger.so run $c; done
FSYRK_B200_LIB=$PWD/profiles/variants/ktrace.so python profiles/ktrace.py cfg2 2>&1 | tail -10
FSYRK_B200_LIB=$PWD/profiles/variants/ktrace.so python profiles/ktrace.py cfg3 2>&1 | tail -6
