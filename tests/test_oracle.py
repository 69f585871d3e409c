"""Pin the C oracle against the reference's own outputs (CPU only).

The golden fixtures were produced by the unmodified reference compiled from
/root/reference (oracle/_ref/ref_driver, tests/golden/make_golden.py).
"""
import numpy as np
import pytest

import oracle_py as orc


def test_random_matrix_stream_matches_reference(golden):
    # random_matrix(f, n, k, seed) (matrix.hpp:411-419): mt19937_64 + libstdc++ uniform_int_distribution
    for case in golden["cases"]:
        if case["mode"] in ("herk", "syrk2"):  # QuadExtField::random_element draws a, then b
            a = orc.random_matrix(case["p"], case["n"], 2 * case["k"], case["seed"]).reshape(case["n"], case["k"], 2)
        else:
            a = orc.random_matrix(case["p"], case["n"], case["k"], case["seed"])
        assert np.array_equal(a, case["A"]), (case["p"], case["n"], case["k"])


def test_mt19937_64_known_value():
    # the C++ standard fixes the 10000th output of default-seeded mt19937_64
    assert int(orc.mt64_stream(5489, 10000)[-1]) == 9981545732273789042


def test_skew_constants_match_reference(golden):
    for p, form, a, b in zip(golden["skew_p"], golden["skew_form"], golden["skew_a"], golden["skew_b"]):
        f, ya, yb, _ = orc.skew(int(p))
        assert (f, ya, yb) == (int(form), int(a), int(b)), int(p)


def test_skew_known_answers():
    # test_fields.cpp:248-292: p=5 -> 2; p=11 -> Pair(1, 3); p=131071 -> pair with a^2+b^2 = -1, ycost 3
    assert orc.skew(5)[:2] == (0, 2)
    assert orc.skew(11)[:3] == (1, 1, 3)
    form, a, b, yc = orc.skew(131071)
    assert form == 1 and (a * a + b * b) % 131071 == 131070 and yc == 3
    # SURVEY §8 constants for the configs
    assert orc.skew(65537)[:2] == (0, 256)
    assert orc.skew(131071)[1:3] == (58294, 93411)
    assert orc.skew(65521)[:2] == (0, 24297)
    assert orc.skew(2147483647)[1:3] == (1008985157, 1682274375)


def test_oracle_matches_reference_outputs(golden):
    for case in golden["cases"]:
        p, a = case["p"], case["A"]
        if case["mode"] in ("herk", "syrk2"):  # F_{p^2}: classical (conjugate) product
            assert orc.lqnr(p) == case["ns"]
            c = orc.fp2_syrk_classical(p, a, case["mode"] == "herk")
            n = case["n"]
            for i in range(n):
                assert np.array_equal(c[i, :i + 1], case["C"][i, :i + 1]), (case["mode"], p, n, case["k"], i)
            continue
        lev = orc.UNLIMITED if case["levels"] is None else case["levels"]
        if case["mode"] == "plain":
            c = orc.syrk_fast(p, a, case["threshold"], lev)
            cls = orc.syrk_classical(p, a)
            assert orc.lower_equal(cls, case["C"]), (p, case["n"], case["k"])
        elif case["mode"] == "acc":
            c = orc.syrk_fast_acc(p, case["alpha"], a, case["beta"], case["C0"], case["threshold"], lev)
        elif case["mode"] == "syrkbd":  # the dense A B A^T restatement (abat_oracle)
            c = orc.abat_classical(p, a, [tuple(int(v) for v in row) for row in case["D"]])
        else:  # schur: Low(C0) - Low(A D A^T)
            x = orc.syrkd(p, a, case["D"], case["threshold"], lev)
            c = case["C0"].copy()
            idx = np.tril_indices(case["n"])
            c[idx] = (c[idx] + np.uint64(p) - x[idx]) % np.uint64(p)
        assert orc.lower_equal(c, case["C"]), (case["mode"], p, case["n"], case["k"])
        assert orc.lower_digest(case["C"]) == case["digest"]


def test_alpha_beta_convention_matches_reference(golden):
    for case in golden["cases"]:
        if case["mode"] == "acc":
            assert orc.alpha_beta(case["p"], case["seed"] + 2) == (case["alpha"], case["beta"])


def test_white_box_identities():
    # test_fast_syrk.cpp:120-190: U3 = C11, U4 = C21, U5 = C22 for one level
    p = 131071
    a = orc.random_matrix(p, 8, 8, 321)
    blk = orc.level_blocks(p, a)
    full = orc.syrk_classical(p, a)
    h = 4
    P1, P2, P3, P4, P5 = (blk[k].astype(object) for k in ("P1", "P2", "P3", "P4", "P5"))
    def sym(x):
        lo = np.tril(x)
        return lo + np.tril(x, -1).T
    U1 = (sym(P1) + sym(P5)) % p
    assert np.array_equal(np.tril((P1 + P2) % p), np.tril(full[:h, :h]))
    assert np.array_equal((U1 + P4 + P3) % p, full[h:, :h])
    assert np.array_equal(np.tril((U1 + P4 + P4.T) % p), np.tril(full[h:, h:]))


@pytest.mark.parametrize("p", [5, 7, 11, 13, 131071, 65537, 2147483647])
def test_nrsyf_and_sqrt(p):
    L = orc.lib()
    for k in range(1, 40):
        r = L.orc_sqrt(p, k)
        if L.orc_legendre(p, k) == 1:
            assert (r * r) % p == k % p and r <= p - r
        elif k % p == 0:
            assert r == 0
        else:
            assert r == (1 << 64) - 1
