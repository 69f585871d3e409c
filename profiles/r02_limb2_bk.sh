# LIMB2 stage geometry: BK = 128 x 3 stages (shipped) vs BK = 64 x 6 / 7 stages
for rep in 1 2; do
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_l2_bk64_s6.so build_variants/lib_l2_bk64_s7.so; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg3', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'], d['roofline']['frac'])"
done
done
