# tile schedule of the persistent product launch: dynamic (atomic counter) vs balanced (static LPT) vs strided
FSYRK_B200_SCHED=dynamic timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
for m in dynamic balanced strided; do
for c in "cfg2 --steps 20" "cfg3 --steps 10" "cfg5 --steps 5" "cfg4 --steps 4" "cfg1 --steps 20"; do
  FSYRK_B200_SCHED=$m timeout 300 python bench.py --config $c --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$m $c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms']['products'], d['roofline']['frac'])"
done
done
done
