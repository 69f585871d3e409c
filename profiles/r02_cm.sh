timeout 600 python -m pytest tests/test_gpu_colmap_fused.py tests/test_gpu_parity.py -x -q -k "fused or syrkbd or golden or syrkd" 2>&1 | tail -15
for v in 0 1; do
  if [ $v = 1 ]; then export FSYRK_B200_NO_CM_FUSE=1; fi
  python bench.py --config cfg5 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nofuse=$v cfg5', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'], d['roofline']['elementwise_hbm'].get('pre'))"
done
