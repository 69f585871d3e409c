for v in build_variants/lib_m17n.so paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_m17n.so paper_2001_04109_b200/libfsyrk_b200.so; do
  for c in "cfg2 --steps 10" "cfg5 --steps 5"; do
  FSYRK_B200_LIB=$v python bench.py --config $c --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'], d['plan']['block_n'])"
  done
done
