"""Per-rank cost of the multi-GPU partition, measured one rank at a time on one GPU.

    python profiles/partition_estimate.py [cfg2] [--ranks 2 4 8]

Each rank's share (fsyrk_b200_syrk_part_dev) is independent (no rank waits on another), so
the N-GPU device time of bench.py --gpus N is the max over ranks of these times; this prints
them next to the single-GPU time, i.e. the strong-scaling speedup before NCCL / launch noise.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2001_04109_b200 as fs  # noqa: E402


def timed(fn, reps=10):
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    for _ in range(3):
        fn()
    ms = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return float(np.median(ms))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="cfg2")
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    p, n, k = c["p"], c["n"], c["k"]
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randint(0, p, (n, k), dtype=torch.int64, device="cuda", generator=g)
    cm = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    pol = fs.RecursionPolicy(c["threshold"], c["levels"])
    s = torch.cuda.current_stream().cuda_stream
    one = timed(lambda: fs.syrk_dev(p, 1, a.data_ptr(), n, k, k, 0, cm.data_ptr(), n, pol, False, s))
    print(json.dumps({"config": args.config, "ranks": 1, "ms": round(one, 4)}))
    for nr in args.ranks:
        per = [timed(lambda r=r: fs.syrk_part_dev(p, 1, a.data_ptr(), n, k, k, 0, cm.data_ptr(), n, pol, r, nr, s))
               for r in range(nr)]
        print(json.dumps({"config": args.config, "ranks": nr, "max_ms": round(max(per), 4),
                          "per_rank_ms": [round(x, 4) for x in per], "speedup": round(one / max(per), 2),
                          "efficiency": round(one / max(per) / nr, 3)}))


if __name__ == "__main__":
    main()
