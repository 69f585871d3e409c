run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 lib=$(basename ${FSYRK_B200_LIB:-default})', d['ms_per_step'], d['roofline']['phase_ms'], d['parity'])"; }
run cfg3
for v in l2bk64s6 l2bk64s5 l2s2; do FSYRK_B200_LIB=$PWD/profiles/variants/$v.so run cfg3; done
