for v in default epw16 epw12 default epw16 epw12; do
  unset FSYRK_B200_LIB; if [ $v != default ]; then export FSYRK_B200_LIB=profiles/variants/$v.so; fi
  for c in cfg2 cfg5; do
    echo "$v $c $(python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"], d["roofline"]["frac"], d["roofline"].get("phase_ms"))')"
  done
done
