# LIMB2 wide-B on CTA pairs (FSYRK_LIMB2_PAIR=1, B planes split across the pair) vs the shipped single-CTA wide-B
V=build_variants/lib_limb2pair.so
FSYRK_B200_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_longk.py -x -q -k "not acceptance" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_longk.py tests/test_gpu_configs.py -x -q -k "not acceptance" 2>&1 | tail -3
for rep in 1 2; do
for v in paper_2001_04109_b200/libfsyrk_b200.so $V; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg3', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'], d['roofline']['frac'], d['plan'].get('terms'))"
done
done
for c in cfg1 cfg2 cfg4 cfg5; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'], d['roofline']['frac'], d.get('launches_per_step'))"
done
python bench.py --config cfg3 --levels 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 depth0', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'], d['roofline']['frac'], d.get('launches_per_step'))"
