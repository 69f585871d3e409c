"""Per-tile timeline of the product kernel's CTA 0 (variant built with -DFSYRK_KTRACE).

    FSYRK_B200_LIB=profiles/variants/ktrace.so python profiles/ktrace.py cfg2
Slots (clock64): 0 MMA warp starts waiting for TMEM, 1 resumes (accumulators free), 2 last
MMA of the tile issued + committed, 3 epilogue warp 2 sees the accumulators, 4 warp 2
released TMEM, 5 warp 9 released TMEM, 6 warp 2 done with the tile.
"""
import ctypes
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
sys.path.insert(0, REPO)
sys.argv = ["run_config.py", cfg, "--iters", "2"]
import runpy  # noqa: E402
runpy.run_path(os.path.join(REPO, "profiles", "run_config.py"), run_name="__main__")
import paper_2001_04109_b200 as fs  # noqa: E402
buf = (ctypes.c_ulonglong * (64 * 8))()
fs.lib().fsyrk_b200_debug_ktrace(buf, 64 * 8)
t = np.array(buf, dtype=np.int64).reshape(64, 8)
t = t[t[:, 1] > 0]
base = t[0, 1]
print("tile  wait->resume  issue(1->2)  mma_done(2->3)  drain(3->4)  drain9(3->5)  epi_total(3->6)  gap(3->next1)")
for i in range(len(t)):
    r = t[i] - base
    nxt = t[i + 1, 1] - t[i, 3] if i + 1 < len(t) else 0
    print(f"{i:3d} {t[i,1]-t[i,0]:10d} {t[i,2]-t[i,1]:10d} {t[i,3]-t[i,2]:12d} {t[i,4]-t[i,3]:10d} {t[i,5]-t[i,3]:10d} "
          f"{t[i,6]-t[i,3]:12d} {nxt:10d}   start={r[1]}")
