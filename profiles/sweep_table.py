"""Summarise profiles/policy_sweep.sh output (JSON lines) as a table."""
import json
import sys

print(f"{'config':6} {'levels':>6} {'ms/step':>9} {'TOPS':>8} {'parity':14} {'products':>9} {'pre':>8} {'post':>8} "
      f"{'convert':>8} {'tensor-frac':>11}")
for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    ph = d["roofline"]["phase_ms"]
    print(f"{d['config']['workload']:6} {str(d['config']['levels']):>6} {d['ms_per_step']:9.4f} "
          f"{d['value'] / 1e3:8.1f} {str(d['parity']):14} {ph['products']:9.4f} {ph['pre']:8.4f} {ph['post']:8.4f} "
          f"{ph['convert']:8.4f} {d['roofline']['frac']:11.3f}")
