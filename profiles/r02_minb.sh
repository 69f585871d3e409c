for v in build_variants/lib_minb3.so build_variants/lib_minb8.so paper_2001_04109_b200/libfsyrk_b200.so; do
  for rep in 1 2; do
  FSYRK_B200_LIB=$v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'])"
  done
done
