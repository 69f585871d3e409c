"""Small host-API calls for compute-sanitizer (memcheck / racecheck) runs: packed and uint32
transfers, pageable and pinned C (duplex accumulate), mirror, syrkd, every digit scheme."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle_py as orc  # noqa: E402
import paper_2001_04109_b200 as fs  # noqa: E402

ok = True
for p in (131071, 65521, 65537, 2147483647, 13):
    f = fs.PrimeField(p)
    for n, k in ((300, 200), (96, 130)):
        a = orc.random_matrix(p, n, k, 3)
        want = orc.syrk_classical(p, a)
        plan = fs.make_syrk_plan(f, fs.RecursionPolicy(16))
        ok &= orc.lower_equal(fs.syrk_fast(f, a, plan), want)
        c = torch.zeros((n, n), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        fs.syrk_fast_acc(f, 3, a, 5, c, plan)
        ok &= orc.lower_equal(c, want * np.uint64(3) % np.uint64(p))
        m = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(16), mirror_output=True))
        ok &= bool(np.array_equal(m, m.T))
        d = orc.random_nonzero(p, k, 4) if p > 3 else None
        if d is not None:
            ok &= orc.lower_equal(fs.syrkd(f, a, d, plan), orc.syrkd(p, a, d, 16))
print("sanitize_small:", "ok" if ok else "MISMATCH")
