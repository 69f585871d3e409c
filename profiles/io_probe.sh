export FSYRK_B200_IO_TRACE=1
timeout 300 python -m pytest tests -m gpu -x -q -k "host or triangular or golden or strided" 2>&1 | tail -2
for up in 0 0.12 0.25; do for dn in 0 0.2 0.35; do
echo "raw up=$up down=$dn"; FSYRK_B200_RAW_UP=$up FSYRK_B200_RAW_DOWN=$dn python profiles/io_probe.py 131071 4096 4096 plain pinned 2>&1 | tail -2
done; done
echo "cfg3 shape duplex"; python profiles/io_probe.py 65521 8192 2048 acc pinned 2>&1 | tail -2
echo "cfg3 shape duplex early"; FSYRK_B200_CIN_EARLY=1 python profiles/io_probe.py 65521 8192 2048 acc pinned 2>&1 | tail -2
echo "cfg3 shape narrow pinned"; FSYRK_B200_HOSTIO=narrow python profiles/io_probe.py 65521 8192 2048 acc pinned 2>&1 | tail -2
echo "cfg3 shape pageable"; python profiles/io_probe.py 65521 8192 2048 acc pageable 2>&1 | tail -2
echo "cfg2 shape pageable"; python profiles/io_probe.py 131071 4096 4096 plain pageable 2>&1 | tail -2
