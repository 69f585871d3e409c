# r02 first verification: GPU tests of the K-chunk drain + multi-GPU library entries, then a
# default bench line (cfg2) and the depth-0 rows.
mkdir -p gpurun_out/r02
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02/bench_default.json 2> gpurun_out/r02/bench_default.err; echo bench rc=$?
cat gpurun_out/r02/bench_default.json
