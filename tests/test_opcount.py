"""OpCount parity with the reference (host only, no device).

tests/golden/opcounts.json holds the OpCount the UNMODIFIED reference accumulated
for 153 calls (tests/golden/make_opcounts.py, oracle/_ref/ref_driver): the count
model's own grid (test_fast_syrk.cpp:202-230), ragged / odd / k > n / Pair-padded
shapes over every skew class, the accumulating form with alpha, beta in {0, 1,
other}, syrkd, syrkbd and F_{p^2}.  The library's tally (csrc/ref_opcount.h), which
every entry point adds to its `ops` argument, must match each one exactly.
"""
import json
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CASES = json.load(open(os.path.join(HERE, "golden", "opcounts.json")))["cases"]
UNL = (1 << 64) - 1


def _ids(c):
    return f"{c['mode']}-p{c['p']}-{c['n']}x{c['k']}-t{c['threshold']}-L{c['levels']}"


@pytest.mark.parametrize("case", CASES, ids=[_ids(c) for c in CASES])
def test_reference_opcount_matches_reference(fsyrk, case):
    pol = fsyrk.RecursionPolicy(case["threshold"], UNL if case["levels"] == "inf" else int(case["levels"]))
    p, n, k, mode = case["p"], case["n"], case["k"], case["mode"]
    if mode == "plain":
        got = fsyrk.reference_opcount(p, n, k, pol)
    elif mode == "acc":
        got = fsyrk.reference_opcount(p, n, k, pol, alpha=case["alpha"], beta=case["beta"])
    elif mode == "schur":  # the reference call is syrkd (its subtraction is not tallied)
        got = fsyrk.reference_opcount(p, n, k, pol, d=case["d"])
    elif mode == "syrkbd":
        bd = fsyrk.BlockDiagonal([fsyrk.Block(bool(t), int(d), int(b), int(g)) for (t, d, b, g) in case["blocks"]])
        got = fsyrk.reference_opcount(p, n, k, pol, blocks=bd)
    else:  # herk / syrk2 over F_{p^2}
        got = fsyrk.reference_opcount(p, n, k, pol, fp2=True)
    assert (got.mults, got.adds) == (case["mults"], case["adds"])


def test_hand_counted_cell(fsyrk):
    # test_fast_syrk.cpp:232-238: n = 4, one level, y = 1 (p = 5) gives 92
    assert fsyrk.reference_opcount(5, 4, 4, fsyrk.RecursionPolicy(2, 1)).total() == 92


def test_large_policy_is_cheap(fsyrk):
    # memoised shape recursion: threshold 2, unlimited levels at cfg4's size
    got = fsyrk.reference_opcount(2147483647, 16384, 16384, fsyrk.RecursionPolicy(2))
    assert got.mults > 0 and got.adds > 0


@pytest.mark.skipif(not os.path.exists(os.path.join(REPO, "oracle", "_ref", "ref_driver")),
                    reason="reference driver not built")
def test_live_reference_counts(fsyrk):
    # a few fresh cases straight from the reference binary (not only the committed fixture)
    for (p, n, k, thr, a, b) in ((131071, 70, 46, 3, 1, 0), (65537, 66, 90, 2, 4, 1), (2147483647, 38, 38, 5, 0, 9)):
        out = json.loads(subprocess.run(
            [os.path.join(REPO, "oracle", "_ref", "ref_driver"), "--p", str(p), "--n", str(n), "--k", str(k),
             "--threshold", str(thr), "--mode", "acc", "--alpha", str(a), "--beta", str(b), "--no-digest"],
            check=True, capture_output=True, text=True).stdout)
        got = fsyrk.reference_opcount(p, n, k, fsyrk.RecursionPolicy(thr), alpha=a, beta=b)
        assert (got.mults, got.adds) == (out["ops_mults"], out["ops_adds"])
