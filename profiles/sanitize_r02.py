"""Small calls through the r02 paths for compute-sanitizer (memcheck / racecheck / synccheck):
the fused subtree prep (2 and 3 levels), the fused two-level post (root and non-root parents),
the low-memory schedule, Winograd levels inside the plan, every digit scheme."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle_py as orc  # noqa: E402
import paper_2001_04109_b200 as fs  # noqa: E402

ok = True
for p in (131071, 65521, 65537, 2147483647, 1000000007, 11):
    f = fs.PrimeField(p)
    for (n, k, thr) in ((256, 256, 64), (256, 128, 32), (128, 128, 16)):
        a = orc.random_matrix(p, n, k, 3)
        want = orc.syrk_classical(p, a)
        for lowmem in (False, True):
            fs.set_low_memory(lowmem)
            plan = fs.make_syrk_plan(f, fs.RecursionPolicy(thr))
            ok &= orc.lower_equal(fs.syrk_fast(f, a, plan), want)
            c = orc.random_matrix(p, n, n, 4)
            c0 = c.copy()
            fs.syrk_fast_acc(f, 3, a, 5, c, plan)
            ok &= orc.lower_equal(c, orc.syrk_classical(p, a, 3, 5, c0))
    fs.set_low_memory(False)
    fs.set_winograd_min(256)
    a = orc.random_matrix(p, 512, 512, 5)
    ok &= orc.lower_equal(fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(64))), orc.syrk_classical(p, a))
    fs.set_winograd_min(16384)
    fs.release_cache()
print("sanitize_r02:", "ok" if ok else "MISMATCH")
