mkdir -p gpurun_out/e2e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e2e/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/e2e/pytest_gpu.log
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e/$c.json 2> gpurun_out/e2e/$c.err; echo "$c rc=$?"
done
FSYRK_B200_HOSTIO=narrow python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e/cfg5_narrow.json 2> gpurun_out/e2e/cfg5_narrow.err; echo "cfg5 narrow rc=$?"
FSYRK_B200_HOSTIO=duplex python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e/cfg3_duplex.json 2> gpurun_out/e2e/cfg3_duplex.err; echo "cfg3 duplex rc=$?"
