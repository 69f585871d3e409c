# LIMB4 wide-B over overlapped accumulators (shipped) vs 16 narrow MMAs (FSYRK_LIMB4_WIDE=0)
timeout 900 python -m pytest tests/test_gpu_longk.py tests/test_gpu_combos.py tests/test_gpu_tree.py tests/test_gpu_lowmem.py tests/test_gpu_wino_plan.py tests/test_gpu_parity.py -x -q -k "not acceptance" 2>&1 | tail -2
for v in paper_2001_04109_b200/libfsyrk_b200.so build_variants/lib_limb4_narrow.so; do
  echo $v; FSYRK_B200_LIB=$v python profiles/generic_primes.py 8192 1 | grep -E '"limb4"|"m31"' | cut -c1-200
  FSYRK_B200_LIB=$v python profiles/generic_primes.py 4096 1 | grep -E '"limb4"' | cut -c1-200
done
