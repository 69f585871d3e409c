./profiles/ubench/ubench_hostio 2>&1 | tail -1
for up in 0.12 0.25 0.4; do for dn in 0 0.2 0.4; do
  echo -n "up=$up down=$dn: "; PROBE_CALLS=8 FSYRK_B200_RAW_UP=$up FSYRK_B200_RAW_DOWN=$dn python profiles/io_probe.py 131071 4096 4096 plain pinned 2>&1 | tail -1 | sed 's/.*ms\/call//' | cut -c1-80
done; done
