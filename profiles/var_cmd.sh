FSYRK_B200_LIB=profiles/variants/ktrace_stg256.so python profiles/ktrace.py cfg2 2>&1 | grep -A8 "^tile" | head -8
for v in default stg256 default stg256; do
  unset FSYRK_B200_LIB; if [ $v != default ]; then export FSYRK_B200_LIB=profiles/variants/$v.so; fi
  for c in cfg2 cfg5; do
    echo "$v $c $(python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"], d["roofline"].get("phase_ms"))')"
  done
done
