# Winograd inside the SYRK plan: the top level's P4 / P3 through the Strassen-Winograd engine
# vs direct tensor-core products, on the configs whose top-level products are large.
# Usage (GPU box): bash profiles/r02_wino_ablation.sh > gpurun_out/r02/wino_ablation.jsonl
cd "$(dirname "$0")/.."
run() {  # label winograd_min config levels steps
  FSYRK_B200_WINOGRAD_MIN=$2 python bench.py --config $3 --levels $4 --threshold 2 --steps $5 --warmup 2 \
      --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'label':'$1','config':'$3','levels':$4,'ms':d['ms_per_step'],'parity':d['parity'],'phase_ms':d['roofline']['phase_ms'],'winograd_groups':d.get('plan',{}).get('winograd_groups')}))"
}
run direct 0 cfg4 1 3
run winograd 8192 cfg4 1 3
run direct 0 cfg4 2 3
run winograd 4096 cfg4 2 3
run direct 0 cfg5 1 5
run winograd 512 cfg5 1 5
run direct 0 cfg3 1 5
run winograd 1024 cfg3 1 5
