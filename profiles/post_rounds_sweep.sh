# root post overlapped with the products (one launch + round counters): product CTAs, rounds
run() { python bench.py --config $1 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 rounds=$FSYRK_B200_POST_ROUNDS ctas=$FSYRK_B200_ROUND_CTAS blocks=$FSYRK_B200_POST_BLOCKS', d['ms_per_step'], d['parity'])"; }
for cfg in cfg5 cfg3; do
  FSYRK_B200_POST_ROUNDS=0 run $cfg
  for r in 8 32; do for c in 148 124 100 88; do
    FSYRK_B200_POST_ROUNDS=$r FSYRK_B200_ROUND_CTAS=$c run $cfg
  done; done
  FSYRK_B200_POST_ROUNDS=16 FSYRK_B200_ROUND_CTAS=100 FSYRK_B200_POST_BLOCKS=400 run $cfg
done
