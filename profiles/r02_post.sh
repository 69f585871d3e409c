for rep in 1 2 3; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['parity'], d['roofline']['phase_ms'])"
done
python bench.py --config cfg5 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'])"
python bench.py --config cfg3 --steps 10 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'])"
