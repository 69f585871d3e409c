# L2 eviction hints on the operand loads of general products (FSYRK_TMA_HINTS=1): cfg4 time and DRAM reads
O=gpurun_out/hints; mkdir -p $O
V=build_variants/lib_hints.so
for rep in 1 2; do
for v in paper_2001_04109_b200/libfsyrk_b200.so $V; do
for c in "cfg4 --steps 4"; do
  FSYRK_B200_LIB=$v timeout 300 python bench.py --config $c --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v $c', d['ms_per_step'], d['parity'], r['phase_ms']['products'])"
done
done
done
for v in paper_2001_04109_b200/libfsyrk_b200.so $V; do
  n=$(basename $v .so)
  FSYRK_B200_LIB=$v ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:modmm --launch-skip 1 -c 1 --csv --log-file $O/dram_$n.csv python profiles/run_config.py cfg4 --iters 2 > /dev/null 2>&1; echo "ncu $n rc=$?"; tail -3 $O/dram_$n.csv | cut -d, -f 5,12-
done
