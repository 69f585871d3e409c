mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu_full2.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02/pytest_gpu_full2.log
FSYRK_B200_BENCH_PART1=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('part1', d['ms_per_step'], d['value'], d['parity'], d['scaling'], d['e2e'])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
