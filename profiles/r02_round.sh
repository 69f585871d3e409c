mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/pytest_gpu_full.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02/pytest_gpu_full.log
bash profiles/r02_wino_ablation.sh > gpurun_out/r02/wino_ablation.jsonl 2>&1; cat gpurun_out/r02/wino_ablation.jsonl
