timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "cfg2 --threshold 1024" "cfg3 --threshold 2" "cfg5 --threshold 2"; do
 for L in 0 1; do
  python bench.py --config $c --levels $L --steps 5 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
 done
done
python bench.py --config cfg1 --threshold 64 --levels 0 --steps 10 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
