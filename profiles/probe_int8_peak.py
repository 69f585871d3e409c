"""Measure the dense int8 tensor-core peak of this B200 (roofline denominator).

cuBLASLt int8 GEMM through torch._int_mm, 8192^3, best of 10 (burst) and a
4-second back-to-back loop (sustained), CUDA events.  Writes
profiles/int8_peak.json (MEASURED_PEAKS.json has no int8 figure).
"""
import json
import os
import time

import torch

N = 8192
a = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
burst = 2 * N ** 3 / (best / 1e3) / 1e12
t0 = time.time()
it = 0
s = torch.cuda.Event(True)
s.record()
while time.time() - t0 < 4.0:
    torch._int_mm(a, b)
    it += 1
e = torch.cuda.Event(True)
e.record()
torch.cuda.synchronize()
sustained = 2 * N ** 3 * it / (s.elapsed_time(e) / 1e3) / 1e12
out = {"int8_tops": round(burst, 1), "int8_tops_sustained": round(sustained, 1),
       "how": "torch._int_mm (cuBLASLt) int8 8192^3, 2*N^3 ops: best of 10 (burst), 4 s back-to-back (sustained)",
       "gpu": torch.cuda.get_device_name()}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "int8_peak.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
