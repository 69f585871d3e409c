for rep in 1 2; do
for e in 0.5 1.1 2.0 3.0; do
  FSYRK_B200_BALANCE_EPI=$e timeout 300 python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('epi=$e cfg2', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'], d['roofline']['frac'])"
done
done
