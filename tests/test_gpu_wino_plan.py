"""Strassen-Winograd general products inside the SYRK plan, against the C oracle.

The reference's level computes P4 and P3 with its Winograd engine
(fast_syrk.hpp:108, 117 -> gemm_winograd_nt_into, winograd.hpp:118-169, 195-202).  The build
runs them as direct tensor-core products by default and switches the top level's pair to
Winograd levels over one grouped tensor-core launch where that pays
(fsyrk_b200_set_winograd_min; the default 16384 is the measured crossover).  Here the
switch is lowered so small shapes take the Winograd path; Low(C) must match the oracle
(not another device path) for plain, accumulating, syrkd, Pair-padded and low-memory calls.
"""
import numpy as np
import pytest

import oracle_py as orc

pytestmark = pytest.mark.gpu


@pytest.fixture
def wino(gpu):
    gpu.release_cache()
    gpu.set_winograd_min(256)
    yield gpu
    gpu.set_winograd_min(16384)
    gpu.set_low_memory(False)
    gpu.release_cache()


# (n, k, threshold): root products h x h x kw with min(h, kw) >= 256 -> Winograd levels
SHAPES = [(512, 512, 64),     # one Winograd level (256 -> 128 base products), deeper recursion direct
          (1024, 512, 128),   # h = 512, kw = 256: one level
          (1024, 1024, 256),  # h = kw = 512: two levels
          (768, 600, 100)]    # kw = 300 (Pair: 300 even, 150 odd -> one level, base k = 150)


@pytest.mark.parametrize("p", [131071, 65521, 65537, 2147483647, 1000000007, 11])
def test_winograd_plan_plain(wino, p):
    fs = wino
    f = fs.PrimeField(p)
    for si, (n, k, thr) in enumerate(SHAPES):
        a = orc.random_matrix(p, n, k, 31 * si + 3)
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(thr)))
        assert fs.last_plan()["winograd_groups"] == 1, (p, n, k, fs.last_plan())
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, n, k, thr)


@pytest.mark.parametrize("p", [131071, 65521, 2147483647])
def test_winograd_plan_acc_syrkd_lowmem(wino, p):
    fs = wino
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p % 1013)
    n, k, thr = 512, 512, 64
    pol = fs.RecursionPolicy(thr)
    a = orc.random_matrix(p, n, k, 17)
    c0 = orc.random_matrix(p, n, n, 18)
    alpha, beta = int(rng.integers(1, p)), int(rng.integers(1, p))
    for lowmem in (False, True):
        fs.set_low_memory(lowmem)
        c = c0.copy()
        fs.syrk_fast_acc(f, alpha, a, beta, c, fs.make_syrk_plan(f, pol))
        plan = fs.last_plan()
        assert plan["winograd_groups"] == 1 and plan["schedule"] == ("low-memory" if lowmem else "wide")
        assert orc.lower_equal(c, orc.syrk_classical(p, a, alpha, beta, c0)), (p, lowmem)
        d = [int(x) for x in rng.integers(1, p, size=k)]
        c = fs.syrkd(f, a, d, fs.make_syrk_plan(f, pol))
        assert orc.lower_equal(c, orc.syrkd(p, a, d, thr)), (p, lowmem)


def test_winograd_off_by_default_below_crossover(gpu):
    fs = gpu
    fs.release_cache()
    f = fs.PrimeField(131071)
    a = orc.random_matrix(131071, 512, 512, 1)
    fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(64)))
    assert fs.last_plan()["winograd_groups"] == 0
