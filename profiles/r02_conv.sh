for rep in 1 2; do
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_conv2.so build_variants/lib_conv3.so; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg5', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'])"
done
done
