mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_lowmem.py tests/test_gpu_wino_plan.py tests/test_gpu_tree.py -x -q > gpurun_out/r02/lowmem_tests.log 2>&1; echo rc=$?; tail -25 gpurun_out/r02/lowmem_tests.log
