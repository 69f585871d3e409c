#!/bin/bash
# Recursion-depth ablation (does the recursion pay on B200?): every config at
# depth 0 (one classical leaf over the whole problem) up to 3 levels, device-resident timing,
# digest-checked.  Usage (GPU box): bash profiles/policy_sweep.sh > gpurun_out/sweep.jsonl
cd "$(dirname "$0")/.."
run() {  # config threshold levels
    python bench.py --config "$1" --threshold "$2" --levels "$3" --steps "${STEPS:-5}" --warmup 3 \
        --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
}
for L in 0 1 2; do run cfg1 64 $L; done
for L in 0 1 2 3; do run cfg2 1024 $L; done
for L in 0 1 2 3; do run cfg3 2 $L; done
for L in 0 1 2 3; do run cfg5 2 $L; done
for L in 0 1 2 3; do STEPS=3 run cfg4 2 $L; done
