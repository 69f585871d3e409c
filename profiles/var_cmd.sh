for c in cfg2 cfg5; do
for v in default p3q6 p4q6 q8 default p3q6 p4q6 q8; do
  if [ $v = default ]; then unset FSYRK_B200_LIB; else export FSYRK_B200_LIB=profiles/variants/$v.so; fi
    echo "$v $c $(python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"], d["roofline"].get("phase_ms"))')"
  done
done
