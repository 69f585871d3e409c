# session-4 verification after the container was re-created: GPU tests, default bench line, per-config lines
mkdir -p gpurun_out/s4
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/s4/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4/bench_default.json 2> gpurun_out/s4/bench_default.err; echo bench rc=$?
cat gpurun_out/s4/bench_default.json
for c in cfg1 cfg3 cfg4 cfg5; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'], d['roofline']['frac'], d.get('launches_per_step'))"
done
