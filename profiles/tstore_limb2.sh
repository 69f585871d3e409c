run() { python bench.py --config $1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 lib=$(basename ${FSYRK_B200_LIB:-default})', d['ms_per_step'], d['roofline']['phase_ms'], d['parity'])"; }
for i in 1 2 3 4; do run cfg3; FSYRK_B200_LIB=$PWD/profiles/variants/notstore2.so run cfg3; done
timeout 600 python -m pytest tests -m gpu -x -q -k "65521 or golden or acceptance" 2>&1 | tail -1
