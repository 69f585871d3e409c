# LIMB2: three overlapped accumulators (FSYRK_LIMB2_OVERLAP=1) vs the shipped four (T00|T01|T10|T11)
V=build_variants/lib_limb2_overlap.so
FSYRK_B200_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_longk.py tests/test_gpu_configs.py -x -q -k "not acceptance" 2>&1 | tail -2
for rep in 1 2; do
for v in paper_2001_04109_b200/libfsyrk_b200.so $V; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg3', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'], d['roofline']['frac'])"
done
done
