"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref/ref_driver).

Run in the build container (needs /root/reference to build ref_driver):
    make -C oracle && python tests/golden/make_golden.py

Writes tests/golden/reference_cases.npz: for every case the reference's
inputs (A, and C0 / D where used) and its output Low(C), plus the case
parameters.  A is the reference's random_matrix(p, n, k, seed); storing it
pins the mt19937_64 + uniform_int_distribution stream as well.
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

# (p, n, k, seed, threshold, levels, mode, mirror)
CASES = []
# oracle batteries over the reference's primes (test_fast_syrk.cpp:71-98, acceptance.cpp:45-74)
_rng = np.random.default_rng(2024)
for p in (5, 13, 131041, 2, 3, 11, 7, 131071, 65537, 65521, 2147483647):
    for t in range(4):
        n = int(_rng.integers(1, 65))
        k = int(_rng.integers(1, 65))
        thr = (2, 8, 14)[t % 3]
        CASES.append((p, n, k, 1000 + t, thr, "inf", "plain", False))
# pair-form padding, classical fallback, wide inputs (test_fast_syrk.cpp:100-118)
CASES += [
    (11, 16, 6, 1, 2, "inf", "plain", False), (11, 32, 10, 2, 2, "inf", "plain", False),
    (11, 6, 6, 3, 2, "inf", "plain", False), (7, 10, 10, 4, 2, "inf", "plain", False),
    (7, 64, 34, 5, 2, "inf", "plain", False), (131071, 8, 32, 1, 2, "inf", "plain", False),
    (131071, 16, 96, 2, 4, "inf", "plain", False), (7, 8, 32, 3, 2, "inf", "plain", False),
    (131071, 64, 64, 321, 4, "1", "plain", False), (131071, 24, 24, 8, 2, "inf", "plain", True),
    (131071, 16, 16, 9, 2, "inf", "plain", False), (2147483647, 48, 40, 11, 4, "inf", "plain", False),
]
# accumulating form (test_fast_syrk.cpp:312-375)
for (p, n, k, s) in ((131071, 33, 20, 55), (131071, 64, 64, 56), (7, 17, 23, 77), (65521, 40, 24, 57),
                     (2147483647, 32, 48, 58)):
    CASES.append((p, n, k, s, 2, "inf", "acc", False))
# syrkd / Schur update (test_scaled_syrk.cpp:59-135)
for (p, n, k, s) in ((131071, 32, 16, 5001), (3, 12, 9, 5002), (13, 20, 7, 5003), (7, 16, 16, 5004),
                     (131071, 48, 31, 5005)):
    CASES.append((p, n, k, s, 2, "inf", "schur", False))

# syrkbd block-diagonal scaling (test_scaled_syrk.cpp:137-205, acceptance.cpp:277-345); D holds the
# blocks as (two, d, beta, gamma) rows
for (p, n, k, s) in ((7, 2, 2, 6001), (13, 5, 5, 6002), (131071, 40, 33, 6003), (65537, 24, 17, 6004),
                     (3, 12, 9, 6005), (11, 30, 12, 6006), (2147483647, 20, 26, 6007), (65521, 64, 48, 6008),
                     (131071, 96, 64, 6009), (5, 9, 14, 6010)):
    CASES.append((p, n, k, s, 2, "inf", "syrkbd", False))

# F_{p^2}: herk_fast (conjugate) and syrk_fast over the quadratic extension (QuadExtField);
# A and C are stored as (rows, cols, 2) arrays of (a, b) pairs
for (p, n, k, s) in ((7, 3, 2, 7001), (13, 20, 11, 7002), (131071, 48, 40, 7003), (65521, 33, 64, 7004),
                     (2147483647, 24, 30, 7005), (11, 64, 17, 7006)):
    CASES.append((p, n, k, s, 4, "inf", "herk", False))
for (p, n, k, s) in ((7, 9, 5, 7101), (131071, 40, 24, 7102), (65537, 30, 30, 7103)):
    CASES.append((p, n, k, s, 4, "inf", "syrk2", False))


def run_case(case, tmp):
    p, n, k, seed, thr, lev, mode, mirror = case
    fa, fc, fc0, fd = (os.path.join(tmp, x) for x in ("a", "c", "c0", "d"))
    cmd = [DRIVER, "--p", str(p), "--n", str(n), "--k", str(k), "--seed", str(seed), "--threshold", str(thr),
           "--levels", lev, "--mode", mode, "--cseed", str(seed + 1), "--abseed", str(seed + 2),
           "--dseed", str(seed + 3), "--out-a", fa, "--out-c", fc, "--out-c0", fc0, "--out-d", fd]
    if mirror:
        cmd.append("--mirror")
    info = json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout)
    if mode in ("herk", "syrk2"):
        return {
            "A": np.fromfile(fa, dtype=np.uint64).reshape(n, k, 2),
            "C": np.fromfile(fc, dtype=np.uint64).reshape(n, n, 2),
            "meta": np.array([p, n, k, seed, thr, -1 if lev == "inf" else int(lev), int(mirror), 1, 0],
                             dtype=np.int64),
            "mode": np.array(mode),
            "digest": np.array(""),
            "ns": np.array(info["non_residue"], dtype=np.uint64),
        }, {"skew_form": "none", "skew_a": 0, "skew_b": 0}
    rec = {
        "A": np.fromfile(fa, dtype=np.uint64).reshape(n, k),
        "C": np.fromfile(fc, dtype=np.uint64).reshape(n, n),
        "meta": np.array([p, n, k, seed, thr, -1 if lev == "inf" else int(lev), int(mirror),
                          info["alpha"], info["beta"]], dtype=np.int64),
        "mode": np.array(mode),
        "digest": np.array(info["digest"]),
    }
    if mode in ("acc", "schur"):
        rec["C0"] = np.fromfile(fc0, dtype=np.uint64).reshape(n, n)
    if mode == "schur":
        rec["D"] = np.fromfile(fd, dtype=np.uint64)
    if mode == "syrkbd":
        rec["D"] = np.fromfile(fd, dtype=np.uint64).reshape(-1, 4)
    return rec, info


def main():
    out = {}
    skews = {}
    with tempfile.TemporaryDirectory() as tmp:
        for i, case in enumerate(CASES):
            rec, info = run_case(case, tmp)
            for key, val in rec.items():
                out[f"c{i:03d}_{key}"] = val
            if info["skew_form"] != "none":
                skews[int(case[0])] = (info["skew_form"], info["skew_a"], info["skew_b"])
    out["ncases"] = np.array(len(CASES))
    primes = sorted(skews)
    out["skew_p"] = np.array(primes, dtype=np.uint64)
    out["skew_form"] = np.array([1 if skews[p][0] == "pair" else 0 for p in primes], dtype=np.int64)
    out["skew_a"] = np.array([skews[p][1] for p in primes], dtype=np.uint64)
    out["skew_b"] = np.array([skews[p][2] for p in primes], dtype=np.uint64)
    path = os.path.join(HERE, "reference_cases.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(CASES)} cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
