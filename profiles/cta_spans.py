"""Per-CTA busy spans of the product kernel (variant built with -DFSYRK_KTRACE): when each
CTA passed its prologue and when its last epilogue warp finished, over the last call.

    FSYRK_B200_LIB=profiles/variants/ktrace.so python profiles/cta_spans.py cfg2
"""
import ctypes
import os
import runpy
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
sys.path.insert(0, REPO)
sys.argv = ["run_config.py", cfg, "--iters", "2"]
runpy.run_path(os.path.join(REPO, "profiles", "run_config.py"), run_name="__main__")
import paper_2001_04109_b200 as fs  # noqa: E402
buf = (ctypes.c_ulonglong * (1024 * 3))()
fs.lib().fsyrk_b200_debug_cta_span(buf, 1024 * 3)
s = np.array(buf, dtype=np.int64).reshape(1024, 3)
s = s[s[:, 0] > 0]
t0 = s[:, 0].min()
start, end, ntile = (s[:, 0] - t0) / 1e3, (s[:, 1] - t0) / 1e3, s[:, 2]
print(f"{cfg}: {len(s)} CTAs; prologue done {start.min():.1f}..{start.max():.1f} us; "
      f"last tile done: min {end.min():.1f} us, median {np.median(end):.1f}, max {end.max():.1f}; "
      f"tiles per CTA {ntile.min()}..{ntile.max()}")
print("finish-time histogram (us):", np.histogram(end, bins=8)[0].tolist(), np.round(np.histogram(end, bins=8)[1], 1).tolist())
