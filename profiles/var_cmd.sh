for c in cfg5; do
for v in pdl pdl; do
  unset FSYRK_B200_NO_PDL FSYRK_B200_LIB
  if [ $v != pdl ]; then export FSYRK_B200_LIB=profiles/variants/$v.so; fi
    echo "$v $c $(python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["parity"])')"
  done
done
