# balanced (LPT) tile schedule of the persistent product launch vs the strided default (FSYRK_B200_BALANCE=0)
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
for b in 1 0; do
for c in "cfg2 --steps 20" "cfg3 --steps 10" "cfg5 --steps 5" "cfg4 --steps 4"; do
  FSYRK_B200_BALANCE=$b timeout 300 python bench.py --config $c --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('balance=$b $c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'], d['roofline']['frac'])"
done
done
done
