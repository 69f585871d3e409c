"""Generate tests/golden/opcounts.json: the UNMODIFIED reference's OpCount tallies.

Run in the build container (needs /root/reference to build ref_driver):
    make -C oracle && python tests/golden/make_opcounts.py

For each case oracle/_ref/ref_driver runs the reference's own entry point
(syrk_fast_into, syrk_fast_acc, syrkd, syrkbd, herk_fast / syrk_fast over
F_{p^2}) on its seeded inputs and prints the OpCount it accumulated
(include/fsyrk/opcount.hpp).  syrkd / syrkbd cases also store D (or the
block list), which decides the column-transform tallies.  The library's
OpCount (csrc/ref_opcount.h) must reproduce every case exactly:
tests/test_opcount.py.
"""
from __future__ import annotations

import json
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(REPO, "oracle", "_ref", "ref_driver")

PRIMES = (2, 3, 5, 7, 11, 13, 19, 23, 65521, 65537, 131071, 998244353, 2147483647)
CASES = []
_rng = np.random.default_rng(77)
# the count model's own grid (test_fast_syrk.cpp:202-230): powers of two, 1-2 levels, threshold 2
for p in (5, 13, 11, 19, 7, 23):
    for n in (4, 8, 16, 32):
        for rec in (1, 2):
            if n >= (2 << rec):
                CASES.append(dict(p=p, n=n, k=n, threshold=2, levels=str(rec), mode="plain"))
# ragged / odd / k > n / Pair padding / Winograd peeling, every skew class
for p in PRIMES:
    for t in range(5):
        n = int(_rng.integers(1, 97))
        k = int(_rng.integers(1, 97))
        thr = int((2, 4, 8, 16, 3)[t])
        lev = ("inf", "1", "2", "inf", "3")[t]
        CASES.append(dict(p=p, n=n, k=k, threshold=thr, levels=lev, mode="plain"))
# wide inputs and deep Winograd engines at threshold 2
CASES += [dict(p=131071, n=24, k=80, threshold=2, levels="inf", mode="plain"),
          dict(p=11, n=64, k=34, threshold=2, levels="inf", mode="plain"),
          dict(p=7, n=96, k=96, threshold=2, levels="inf", mode="plain"),
          dict(p=65537, n=128, k=128, threshold=2, levels="inf", mode="plain"),
          dict(p=2147483647, n=100, k=62, threshold=3, levels="inf", mode="plain")]
# accumulating form: alpha / beta classes 0, 1, other
for (p, n, k, a, b) in ((131071, 33, 20, 5, 3), (131071, 64, 64, 1, 1), (7, 17, 23, 0, 4), (65521, 40, 24, 2, 0),
                        (2147483647, 32, 48, 9, 1), (11, 48, 48, 1, 6), (5, 30, 44, 0, 0), (13, 64, 16, 3, 1),
                        (998244353, 50, 50, 7, 8), (3, 36, 36, 2, 2)):
    for thr in (2, 8):
        CASES.append(dict(p=p, n=n, k=k, threshold=thr, levels="inf", mode="acc", alpha=a, beta=b))
# syrkd (schur mode tallies the reference's syrkd call only) and syrkbd
for (p, n, k, s) in ((131071, 32, 16, 5001), (3, 12, 9, 5002), (13, 20, 7, 5003), (7, 16, 16, 5004),
                     (131071, 48, 31, 5005), (65537, 40, 33, 5006), (2147483647, 24, 25, 5007)):
    CASES.append(dict(p=p, n=n, k=k, threshold=2, levels="inf", mode="schur", dseed=s))
for (p, n, k, s) in ((131071, 24, 16, 71), (11, 20, 13, 72), (7, 32, 9, 73), (65521, 16, 20, 74)):
    CASES.append(dict(p=p, n=n, k=k, threshold=2, levels="inf", mode="syrkbd", dseed=s))
# F_{p^2}
for (p, n, k) in ((7, 16, 12), (11, 20, 20), (131071, 24, 9), (13, 32, 32), (3, 9, 14)):
    for mode in ("herk", "syrk2"):
        CASES.append(dict(p=p, n=n, k=k, threshold=2, levels="inf", mode=mode))


def run(case, tmp):
    cmd = [DRIVER, "--p", str(case["p"]), "--n", str(case["n"]), "--k", str(case["k"]),
           "--threshold", str(case["threshold"]), "--levels", case["levels"], "--mode", case["mode"], "--no-digest"]
    if case["mode"] == "acc":
        cmd += ["--alpha", str(case["alpha"]), "--beta", str(case["beta"])]
    dpath = os.path.join(tmp, "d.bin")
    if case["mode"] in ("schur", "syrkbd"):
        cmd += ["--dseed", str(case["dseed"]), "--out-d", dpath]
    out = json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout)
    rec = dict(case)
    rec["mults"] = out["ops_mults"]
    rec["adds"] = out["ops_adds"]
    if case["mode"] == "schur":
        rec["d"] = np.fromfile(dpath, dtype=np.uint64).tolist()
    elif case["mode"] == "syrkbd":
        rec["blocks"] = np.fromfile(dpath, dtype=np.uint64).reshape(-1, 4).tolist()  # (two, d, beta, gamma)
    return rec


def main():
    with tempfile.TemporaryDirectory() as tmp:
        recs = [run(c, tmp) for c in CASES]
    with open(os.path.join(HERE, "opcounts.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_opcounts.py (oracle/_ref/ref_driver, reference sources)",
                   "cases": recs}, f, indent=0)
    print(len(recs), "cases")


if __name__ == "__main__":
    main()
