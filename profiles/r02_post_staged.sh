# single-level / root post: second-round loads staged by cp.async (shipped) vs loaded after the barrier
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2 3; do
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_post_unstaged.so; do
for c in "cfg2 --steps 20" "cfg3 --steps 10" "cfg5 --steps 4" "cfg1 --steps 20"; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config $c --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $c', d['ms_per_step'], d['parity'], r['phase_ms']['post'], r['elementwise_hbm']['post']['frac'])"
done
done
done
