python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'], d['launches_per_step'])"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02/launches_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
FSYRK_B200_TRACE=1 python profiles/run_config.py cfg1 --iters 3 2>&1 | tail -12
