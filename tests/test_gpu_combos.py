"""Seeded combinations of the plan's switches against the C oracle.

Every switch changes how a call is executed, never its result (exact arithmetic): the fused
subtree prep (automatic for complete uniform trees), the low-memory schedule
(fsyrk_b200_set_low_memory), Strassen-Winograd levels for the top level's products
(fsyrk_b200_set_winograd_min), and the entry point (plain, accumulating, syrkd Schur form).
Random shapes (odd, ragged, k > n, Pair padding), primes over every digit scheme and both skew
forms, and recursion policies; Low(C) must equal the oracle's in every combination.
"""
import os

import numpy as np
import pytest

import oracle_py as orc

pytestmark = pytest.mark.gpu

PRIMES = [131071, 65537, 65521, 2147483647, 998244353, 1000000007, 11, 13, 7]


@pytest.fixture
def switches(gpu):
    yield gpu
    gpu.set_low_memory(False)
    gpu.set_winograd_min(16384)
    gpu.release_cache()


SEEDS = int(os.environ.get("FSYRK_COMBO_SEEDS", "6"))  # stress runs: FSYRK_COMBO_SEEDS=60


@pytest.mark.parametrize("seed", range(SEEDS))
def test_switch_combinations(switches, seed):
    fs = switches
    rng = np.random.default_rng(1000 + seed)
    for case in range(10):
        p = int(rng.choice(PRIMES))
        f = fs.PrimeField(p)
        shape = rng.integers(4)
        if shape == 0:    # complete uniform tree (fused prep), power-of-two sizes
            n = int(rng.choice([128, 256, 512]))
            k = n // int(rng.choice([1, 2]))
        elif shape == 1:  # ragged / odd
            n, k = int(rng.integers(1, 400)), int(rng.integers(1, 400))
        elif shape == 2:  # k > n (split on k)
            n = int(rng.integers(16, 200))
            k = n + int(rng.integers(1, 300))
        else:             # Pair padding: kh odd
            n = 2 * int(rng.integers(20, 150))
            k = 2 * (2 * int(rng.integers(5, 60)) + 1)
        thr = int(rng.choice([2, 16, 32, 64, 1000]))
        lev = int(rng.choice([1, 2, 3, 1 << 40]))
        pol = fs.RecursionPolicy(thr, (1 << 64) - 1 if lev == 1 << 40 else lev)
        lowmem = bool(rng.integers(2))
        wmin = int(rng.choice([16384, 256]))
        fs.set_low_memory(lowmem)
        fs.set_winograd_min(wmin)
        mode = int(rng.integers(3))
        a = orc.random_matrix(p, n, k, int(rng.integers(1 << 62)))
        plan = fs.make_syrk_plan(f, pol)
        tag = (seed, case, p, n, k, thr, lev, lowmem, wmin, mode)
        if mode == 0:
            c = fs.syrk_fast(f, a, plan)
            assert orc.lower_equal(c, orc.syrk_classical(p, a)), tag
        elif mode == 1:
            c0 = orc.random_matrix(p, n, n, 7)
            alpha, beta = int(rng.integers(p)), int(rng.integers(p))
            c = c0.copy()
            fs.syrk_fast_acc(f, alpha, a, beta, c, plan)
            assert orc.lower_equal(c, orc.syrk_classical(p, a, alpha, beta, c0)), tag
        elif p != 2:
            d = [int(x) for x in rng.integers(1, p, size=k)]
            c0 = orc.random_matrix(p, n, n, 9)
            c = c0.copy()
            fs.syrkd(f, a, d, plan, alpha=p - 1, beta=1, c=c)
            x = orc.syrkd(p, a, d, thr, pol.max_levels)
            want = (c0 + (np.uint64(p) - x) % np.uint64(p)) % np.uint64(p)
            assert orc.lower_equal(c, want), tag
