export FSYRK_B200_IO_TRACE=1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for pk in 1 0; do
echo "cfg2 pack=$pk"; FSYRK_B200_PACK=$pk python profiles/io_probe.py 131071 4096 4096 plain pinned 2>&1 | tail -2
echo "cfg2 pack=$pk raw0"; FSYRK_B200_RAW_UP=0 FSYRK_B200_PACK=$pk python profiles/io_probe.py 131071 4096 4096 plain pinned 2>&1 | tail -2
echo "cfg2 pack=$pk raw25"; FSYRK_B200_RAW_UP=0.25 FSYRK_B200_RAW_DOWN=0.2 FSYRK_B200_PACK=$pk python profiles/io_probe.py 131071 4096 4096 plain pinned 2>&1 | tail -2
echo "cfg3 pack=$pk narrow"; FSYRK_B200_HOSTIO=narrow FSYRK_B200_PACK=$pk python profiles/io_probe.py 65521 8192 2048 acc pinned 2>&1 | tail -2
echo "cfg3 pack=$pk duplex"; FSYRK_B200_PACK=$pk python profiles/io_probe.py 65521 8192 2048 acc pinned 2>&1 | tail -2
done
