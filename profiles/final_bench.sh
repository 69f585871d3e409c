mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/final/pytest_gpu.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/reference_cfg2.json 2> gpurun_out/final/reference_cfg2.err; echo "ref rc=$?"
python bench.py > gpurun_out/final/default.json 2> gpurun_out/final/default.err; echo "default rc=$?"
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final/$c.json 2> gpurun_out/final/$c.err; echo "$c rc=$?"
done
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
