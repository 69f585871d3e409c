export FSYRK_B200_IO_TRACE=1
timeout 600 python -m pytest tests -m gpu -x -q -k "host_io or triangular or cfg5 or cfg3 or syrkd" 2>&1 | tail -2
for f in 0 0.25 0.4 0.55 0.7; do
  echo "frac=$f"; FSYRK_B200_DUPLEX_PACKED=$f python profiles/io_probe.py 131071 16384 1024 acc pinned 2>&1 | tail -2
done
for f in 0 0.4 0.55; do
  FSYRK_B200_DUPLEX_PACKED=$f python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 frac=$f e2e', d['e2e'])"
done
