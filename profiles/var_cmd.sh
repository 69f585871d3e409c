timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for v in default m31bk32 default m31bk32; do
  unset FSYRK_B200_LIB; if [ $v != default ]; then export FSYRK_B200_LIB=profiles/variants/$v.so; fi
  for c in cfg4; do
    echo "$v $c $(python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"], d["roofline"]["frac"], d["roofline"].get("phase_ms"), d["clocks"]["sm_mhz"])')"
  done
done
