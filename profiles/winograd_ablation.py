"""Strassen-Winograd levels over the tensor-core product on the B200 (SURVEY 8f rank 2 ablation).

    python profiles/winograd_ablation.py [--p 131071] [--sizes 4096 8192] [--levels 0 1 2 3]

Times fsyrk_b200_gemm_winograd_nt_dev (device-resident uint64 A, B, C; CUDA events, L2 flushed
between runs) and checks every depth against depth 0 (exact products are bit-identical).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04109_b200 as fs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=131071)
    ap.add_argument("--sizes", type=int, nargs="+", default=[4096, 8192])
    ap.add_argument("--levels", type=int, nargs="+", default=[0, 1, 2, 3])
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    p = args.p
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    for n in args.sizes:
        g = torch.Generator(device="cuda").manual_seed(n)
        a = torch.randint(0, p, (n, n), dtype=torch.int64, device="cuda", generator=g)
        b = torch.randint(0, p, (n, n), dtype=torch.int64, device="cuda", generator=g)
        ref = None
        for lev in args.levels:
            c = torch.zeros((n, n), dtype=torch.int64, device="cuda")
            pol = fs.RecursionPolicy(256, lev)
            s = torch.cuda.current_stream().cuda_stream
            fs.gemm_winograd_nt_dev(p, a.data_ptr(), n, n, n, b.data_ptr(), n, n, c.data_ptr(), n, pol, s)
            torch.cuda.synchronize()
            if ref is None:
                ref = c.clone()
            same = bool(torch.equal(c, ref))
            ms = []
            for _ in range(args.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fs.gemm_winograd_nt_dev(p, a.data_ptr(), n, n, n, b.data_ptr(), n, n, c.data_ptr(), n, pol, s)
                e1.record()
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            t = float(np.median(ms))
            print(json.dumps({"n": n, "levels": lev, "ms": round(t, 3), "effective_tops": round(2 * n ** 3 / t / 1e9, 1),
                              "equal_to_direct": same}))


if __name__ == "__main__":
    main()
