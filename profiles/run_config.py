"""Run one bench config's hot-path call a few times on cuda:0 (for ncu / trace captures).

    python profiles/run_config.py cfg2 [--iters 4]
    FSYRK_B200_TRACE=1 python profiles/run_config.py cfg2        # per-phase device timeline
    ncu --set full -k regex:modmm --launch-skip 3 -c 1 ... python profiles/run_config.py cfg2

Inputs are generated on the device (device-resident, like bench.py's `value`); no
parity check here (bench.py and the tests do that).
"""
import argparse
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import paper_2001_04109_b200 as fs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="cfg2")
    ap.add_argument("--iters", type=int, default=4)
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    p, n, k = c["p"], c["n"], c["k"]
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randint(0, p, (n, k), dtype=torch.int64, device="cuda", generator=g)
    cm = torch.randint(0, p, (n, n), dtype=torch.int64, device="cuda", generator=g)
    pol = fs.RecursionPolicy(c["threshold"], c["levels"])
    alpha, beta, d = 1, 0, None
    if c["mode"] == "acc":
        alpha, beta = 12345 % p, 678 % p
    elif c["mode"] == "schur":
        alpha, beta = p - 1, 1
        d = np.random.default_rng(2).integers(1, p, size=k, dtype=np.uint64)
    s = torch.cuda.current_stream().cuda_stream
    for i in range(args.iters):
        if i == args.iters - 1:
            print("---- last call", file=sys.stderr)
        fs.syrk_dev(p, alpha, a.data_ptr(), n, k, k, beta, cm.data_ptr(), n, pol, False, s, d=d)
        torch.cuda.synchronize()
    print(f"{args.config}: {args.iters} calls ok")


if __name__ == "__main__":
    main()
