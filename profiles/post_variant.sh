run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 lib=$FSYRK_B200_LIB', d['ms_per_step'], d['roofline']['phase_ms'], d['parity'])"; }
for lib in paper_2001_04109_b200/libv_mb3.so paper_2001_04109_b200/libv_mb4.so; do
  for c in cfg2 cfg3 cfg5 cfg4; do FSYRK_B200_LIB=$PWD/$lib run $c; done
done
