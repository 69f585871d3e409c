run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 lib=$(basename ${FSYRK_B200_LIB:-default})', d['ms_per_step'], d['roofline']['phase_ms'], d['parity'])"; }
for c in cfg2 cfg5 cfg3; do run $c; FSYRK_B200_LIB=$PWD/profiles/variants/poststream.so run $c; done
