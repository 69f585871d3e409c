"""Device-resident timing of the hot path over generic primes (the LIMB3 / LIMB4 schemes no
BASELINE config exercises at size): effective TOPS n^2 k / t, phase split, plan.

    python profiles/generic_primes.py [n] [levels]
"""
import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2001_04109_b200 as fs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 1
k = n
PRIMES = [65521, 131071, 8380417, 16777213, 998244353, 1000000007, 2147483629, 2147483647]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for p in PRIMES:
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randint(0, p, (n, k), dtype=torch.int64, device="cuda", generator=g)
    c = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    pol = fs.RecursionPolicy(2, levels)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        fs.syrk_dev(p, 1, a.data_ptr(), n, k, k, 0, c.data_ptr(), n, pol, False, s)
    torch.cuda.synchronize()
    t = []
    for _ in range(8):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fs.syrk_dev(p, 1, a.data_ptr(), n, k, k, 0, c.data_ptr(), n, pol, False, s)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    ms = sorted(t)[len(t) // 2]
    fs.set_phase_timing(True)
    fs.syrk_dev(p, 1, a.data_ptr(), n, k, k, 0, c.data_ptr(), n, pol, False, s)
    torch.cuda.synchronize()
    ph = fs.last_phase_ms()
    fs.set_phase_timing(False)
    plan = fs.last_plan()
    print(json.dumps({"p": p, "n": n, "levels": levels, "ms": round(ms, 4), "tops": round(n * n * k / ms / 1e9, 1),
                      "scheme": plan.get("scheme"), "terms": plan.get("terms"), "block_n": plan.get("block_n"),
                      "phase_ms": ph}))
