"""Host-API (e2e) timing probe: pinned vs pageable caller buffers, per-phase host timings
(FSYRK_B200_IO_TRACE=1 prints one [io] line per call to stderr)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04109_b200 as fs  # noqa: E402


def pinned(shape):
    return torch.empty(shape, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)


def main():
    p, n, k, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    pin = len(sys.argv) > 5 and sys.argv[5] == "pinned"
    f = fs.PrimeField(p)
    rng = np.random.default_rng(1)
    a = pinned((n, k)) if pin else np.empty((n, k), dtype=np.uint64)
    a[:] = rng.integers(0, p, size=(n, k), dtype=np.uint64)
    c = pinned((n, n)) if pin else np.empty((n, n), dtype=np.uint64)
    c[:] = 1
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(512, 1))
    ts = []
    for it in range(int(os.environ.get('PROBE_CALLS', '6'))):
        t0 = time.perf_counter()
        if mode == "plain":
            fs.syrk_fast_into(f, a, c, plan)
        else:
            fs.syrk_fast_acc(f, 3, a, 5, c, plan)
        ts.append(time.perf_counter() - t0)
    print(f"p={p} n={n} k={k} {mode} pinned={pin}: ms/call", [round(t * 1e3, 3) for t in ts],
          "bytes", fs.last_transfer_bytes(), flush=True)


if __name__ == "__main__":
    main()
