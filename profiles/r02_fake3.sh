# Timing-only: M17 products with only the 3 digit planes of A loaded (FSYRK_M17_FAKE3; results wrong by design)
for rep in 1 2; do
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_fake3.so; do
for c in cfg2 cfg5; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v $c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'])"
done
done
done
