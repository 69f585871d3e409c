run() { python bench.py --config $1 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 lib=$(basename ${FSYRK_B200_LIB:-default})', d['ms_per_step'], d['roofline']['phase_ms']['products'], d['clocks']['sm_mhz'], d['parity'])"; }
for i in 1 2 3; do run cfg4; FSYRK_B200_LIB=$PWD/profiles/variants/m31pair.so run cfg4; done
FSYRK_B200_LIB=$PWD/profiles/variants/m31pair.so timeout 600 python -m pytest tests -m gpu -x -q -k "2147483647 or golden or gemm" 2>&1 | tail -2
