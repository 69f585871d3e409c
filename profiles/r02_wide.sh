timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_longk.py tests/test_gpu_combos.py tests/test_gpu_configs.py -x -q -k "not acceptance" 2>&1 | tail -3
for rep in 1 2; do
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_limb2narrow.so; do
  FSYRK_B200_LIB=$v python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg3', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'], d['roofline']['frac'], d['plan'].get('terms'))"
done
done
