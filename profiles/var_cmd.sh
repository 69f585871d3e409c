python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FSYRK_B200_LIB=profiles/variants/m17_bn80_s3.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in default m17_bn80_s3 m17_bn80_s4 m17_bn64_s4; do
  if [ $v = default ]; then unset FSYRK_B200_LIB; else export FSYRK_B200_LIB=profiles/variants/$v.so; fi
  for c in cfg2 cfg5; do
    echo "$v $c $(python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"], d["roofline"]["frac"], d.get("phase_ms"))')"
  done
done
