run() { python bench.py --config $1 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 group=$FSYRK_B200_GROUP_ROWS', d['ms_per_step'], d['roofline']['phase_ms']['products'], d['clocks'], d['parity'])"; }
for g in 0 12 6 20; do FSYRK_B200_GROUP_ROWS=$g run cfg4; done
for g in 0 12; do for c in cfg2 cfg3 cfg5; do FSYRK_B200_GROUP_ROWS=$g run $c; done; done
FSYRK_B200_GROUP_ROWS=12 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:modmm --launch-skip 1 -c 1 python profiles/run_config.py cfg4 --iters 2 2>&1 | grep -E "dram__|gpu__time" 
