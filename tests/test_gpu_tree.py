"""Fused subtree pre-additions (prep_tree_kernel) against the C oracle.

Plans whose tree is complete and uniform below the root (D = 2 or 3 levels, every
level unpadded, all leaves at depth D; fast_syrk.hpp:135-157 decides the shape) run
all pre-additions in one launch from the caller's A.  These shapes cover every
digit scheme and both skew forms (ScalarRoot for p = 1 mod 4, Pair otherwise,
skew.hpp:66-73), plus the accumulating form, extreme residues and non-canonical
inputs; each plan is checked to have taken the fused path.
"""
import numpy as np
import pytest

import oracle_py as orc

pytestmark = pytest.mark.gpu

PRIMES = [131071, 65537, 65521, 2147483647, 998244353, 1000000007, 11, 13]
# (n, k, threshold, fused): tree depth D, and whether the one-launch path applies
SHAPES = [(1024, 1024, 256, True),  # D = 3, 128 x 128 leaves: several CTAs per leaf row
          (256, 256, 64, True),    # D = 3
          (128, 128, 32, True),    # D = 3
          (256, 128, 32, True),    # D = 3, k < n
          (208, 128, 48, True),    # D = 2, 52 x 32 leaves
          (200, 120, 40, False),   # D = 2, 50 x 30 leaves: 30 columns are not 4-aligned -> per-depth
          (96, 160, 24, False)]    # k > n: split on k first (not a uniform tree)


@pytest.mark.parametrize("p", PRIMES)
def test_tree_prep_plain(gpu, p):
    fs = gpu
    f = fs.PrimeField(p)
    for si, (n, k, thr, fused) in enumerate(SHAPES):
        a = orc.random_matrix(p, n, k, 1000 * si + 7)
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(thr)))
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, n, k, thr)
        if fused:  # uniform tree: one pre-addition launch
            assert fs.last_launch_counts()["pre"] == 1, (p, n, k, fs.last_launch_counts())


@pytest.mark.parametrize("p", [131071, 65521, 2147483647, 1000000007])
def test_tree_prep_accumulate(gpu, p):
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p % 1000)
    n, k = 256, 256
    a = orc.random_matrix(p, n, k, 99)
    c0 = orc.random_matrix(p, n, n, 98)
    alpha, beta = int(rng.integers(1, p)), int(rng.integers(1, p))
    c = c0.copy()
    fs.syrk_fast_acc(f, alpha, a, beta, c, fs.make_syrk_plan(f, fs.RecursionPolicy(64)))
    assert orc.lower_equal(c, orc.syrk_classical(p, a, alpha, beta, c0))


def test_tree_prep_extreme_and_noncanonical(gpu):
    fs = gpu
    for p in (131071, 65537, 2147483647):
        f = fs.PrimeField(p)
        for val in (p - 1, p // 2, p // 2 + 1):
            a = np.full((128, 128), val, dtype=np.uint64)
            c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(32)))
            assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, val)
        # non-canonical entries (>= p, >= 2^31) are reduced on the way in
        rng = np.random.default_rng(5)
        a = rng.integers(0, 1 << 63, size=(128, 128), dtype=np.uint64)
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(32)))
        assert orc.lower_equal(c, orc.syrk_classical(p, a % np.uint64(p))), p


@pytest.mark.parametrize("p", [131071, 65521, 2147483647, 1000000007])
def test_fused_two_level_post(gpu, p):
    # three-level uniform trees run the two deepest post-addition levels as one launch
    # (post2_kernel): the deepest nodes' X stay in shared memory; plain and accumulating forms
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p % 101)
    for (n, k, thr) in ((1024, 1024, 256), (256, 256, 64), (512, 256, 64)):
        a = orc.random_matrix(p, n, k, n + k + 1)
        plan = fs.make_syrk_plan(f, fs.RecursionPolicy(thr))
        c = fs.syrk_fast(f, a, plan)
        assert fs.last_plan()["post2"] == 1, (p, n, k, fs.last_plan())
        assert fs.last_launch_counts()["post"] == 2, fs.last_launch_counts()
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, n, k)
        c0 = orc.random_matrix(p, n, n, 3)
        alpha, beta = int(rng.integers(1, p)), int(rng.integers(1, p))
        c = c0.copy()
        fs.syrk_fast_acc(f, alpha, a, beta, c, plan)
        assert orc.lower_equal(c, orc.syrk_classical(p, a, alpha, beta, c0)), (p, n, k, "acc")
