for t in 1 0; do
 for c in "cfg4 --levels 2 --threshold 2 --steps 3" "cfg2 --steps 10"; do
  FSYRK_B200_TREE_PREP=$t python bench.py --config $c --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tree=$t', '$c', d['ms_per_step'], d['parity'], d['roofline']['phase_ms'])"
 done
done
python -m pytest tests/test_gpu_tree.py -q -x 2>&1 | tail -1
