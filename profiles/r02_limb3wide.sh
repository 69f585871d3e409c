# LIMB3 wide-B over overlapped accumulators, 80-column tiles (shipped) vs 9 narrow MMAs on 96-column tiles (FSYRK_LIMB3_WIDE=0)
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_limb3_narrow.so; do
  echo $v; FSYRK_B200_LIB=$v python profiles/generic_primes.py 8192 1 | grep -E '"limb3"' | cut -c1-230
  FSYRK_B200_LIB=$v python profiles/generic_primes.py 4096 1 | grep -E '"limb3"' | cut -c1-230
  for rep in 1 2; do FSYRK_B200_LIB=$v python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg1', d['ms_per_step'], d['parity'], r['phase_ms'], r['frac'])"; done
done
