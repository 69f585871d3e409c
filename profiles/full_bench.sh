# full bench lines for every config (device value, roofline, cpu baseline, e2e, clocks) + reference arm
mkdir -p gpurun_out/bench
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench/$c.json 2> gpurun_out/bench/$c.err
  echo "$c rc=$?"
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench/reference_cfg2.json 2> gpurun_out/bench/reference_cfg2.err
echo "ref rc=$?"
python bench.py > gpurun_out/bench/default.json 2> gpurun_out/bench/default.err
echo "default rc=$?"
