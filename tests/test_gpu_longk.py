"""Exactness at any inner dimension, and the LIMB4 digit scheme.

The reference accumulates every dot product in `unsigned __int128` and accepts any k
(proj/include/fsyrk/matrix.hpp:144-160); the device kernel's int32 accumulators are exact only
up to `modmm_k_limit` (tc_modmm.cu), so the product kernel drains them mod p every chunk of at
most that many K (tc_modmm_kernel.cuh, K chunks).  These cases sit just above each scheme's
bound, use the largest digits everywhere (all p - 1) and random mixes, and cover LIMB4 (every
prime in (2^24, 2^31 - 1)) through every path: battery, extreme values, leaves, levels.
All bit-exact against the C oracle."""
import numpy as np
import pytest

import oracle_py as orc

pytestmark = pytest.mark.gpu

UNL = (1 << 64) - 1
LIMB4_PRIMES = [998244353, 1000000007, 2147483629, 16777259]


def _k_limit(p):
    """modmm_k_limit (tc_modmm.cu) restated: the K bound of each digit scheme."""
    i32 = (1 << 31) - 1
    if p == 131071:
        return i32 // (3 * 126 * 63)
    if p == 2147483647:
        return 0xFFFFFFFF // (5 * 255 * 255)
    L = 2 if p <= 65536 else 3 if p <= 16777216 else 4
    return min(i32 // (L * 16384), (1 << 62) // (L * L * 16384 * (p // 2 + 1)))


def _gemm_check(fs, p, m, n, k, extreme):
    f = fs.PrimeField(p)
    if extreme:
        a = np.full((m, k), p - 1, dtype=np.uint64)
        b = np.full((n, k), p - 1, dtype=np.uint64)
    else:
        a = orc.random_matrix(p, m, k, 5)
        b = orc.random_matrix(p, n, k, 6)
        a[:, ::3] = p - 1
        b[:, 1::4] = p // 2  # balanced-digit window edge
    c = fs.gemm_nt(f, a, b)
    full = orc.syrk_classical(p, np.vstack([a, b]))
    assert np.array_equal(c, full[m:, :m].T), (p, m, n, k, extreme)


@pytest.mark.parametrize("p", [2147483647, 131071, 65521, 65537, 998244353, 2147483629])
def test_general_product_above_k_limit(gpu, p):
    # K just above the scheme's int32 bound: two (or three) exact chunks per output tile
    lim = _k_limit(p)
    for k, extreme in ((lim + 300, True), (2 * lim + 129, False)):
        _gemm_check(gpu, p, 130, 70, k, extreme)


@pytest.mark.parametrize("p", [2147483647, 2147483629, 131071])
def test_odd_leaf_above_k_limit(gpu, p):
    # an odd n forces a classical leaf over the whole k (fast_syrk.hpp:139): n = 63 with k above
    # the bound (p = 2^31 - 1, n = 63, k = 13500 was rejected with EINVAL)
    fs = gpu
    f = fs.PrimeField(p)
    k = _k_limit(p) + 290
    for extreme in (True, False):
        a = np.full((63, k), p - 1, dtype=np.uint64) if extreme else orc.random_matrix(p, 63, k, 17)
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(8)))
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, extreme)
        # accumulating form through the same chunked leaf
        c0 = orc.random_matrix(p, 63, 63, 18)
        c = c0.copy()
        fs.syrk_fast_acc(f, 3, a, p - 2, c, fs.make_syrk_plan(f, fs.RecursionPolicy(8)))
        want = orc.syrk_classical(p, a)
        idx = np.tril_indices(63)
        exp = [(int(w) * 3 + int(x) * (p - 2)) % p for w, x in zip(want[idx], c0[idx])]
        assert np.array_equal(c[idx], np.array(exp, dtype=np.uint64))


def test_depth0_leaf_above_k_limit_even_shape(gpu):
    # levels = 0: the whole problem is one leaf SYRK with k above the M31 bound (and even, so a
    # level would otherwise be possible); lower tiles of the SYRK take the chunked epilogue too
    fs = gpu
    p = 2147483647
    f = fs.PrimeField(p)
    n, k = 300, 26500
    a = orc.random_matrix(p, n, k, 23)
    a[::5, :] = p - 1
    c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(2, 0)))
    assert orc.lower_equal(c, orc.syrk_classical(p, a))


@pytest.mark.parametrize("p", [2147483647, 2147483629])
def test_level_with_kw_above_k_limit(gpu, p):
    # one recursion level whose general products P3, P4 (h x h x kw) and leaf SYRKs have an inner
    # dimension above the bound: n = k = 2 kw with kw = limit + 128.  A full oracle SYRK at this size
    # is too slow, so: 384 sampled entries recomputed exactly (oracle __int128 dots), and the
    # lower-triangle digest must equal the depth-0 (single chunked leaf) result's.
    fs = gpu
    torch = pytest.importorskip("torch")
    f = fs.PrimeField(p)
    kw = _k_limit(p) + 128
    kw += kw % 2
    n = k = 2 * kw
    a = orc.random_matrix(p, n, k, 29)
    a_dev = torch.from_numpy(a.view(np.int64)).cuda()
    outs = []
    for levels in (1, 0):
        c_dev = torch.zeros((n, n), dtype=torch.int64, device="cuda")
        fs.syrk_dev(p, 1, a_dev.data_ptr(), n, k, k, 0, c_dev.data_ptr(), n, fs.RecursionPolicy(2, levels), False,
                    torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        plan = fs.last_plan()
        if levels == 1:
            assert plan["gemm_groups"][0]["kw"] > _k_limit(p), plan
        outs.append(torch.tril(c_dev).cpu().numpy().view(np.uint64))
        del c_dev
    assert np.array_equal(outs[0], outs[1])
    rng = np.random.default_rng(31)
    for _ in range(384):
        i = int(rng.integers(n))
        j = int(rng.integers(i + 1))
        assert int(outs[0][i, j]) == orc.dot_mod(p, a[i], a[j]), (i, j)


@pytest.mark.parametrize("p", LIMB4_PRIMES)
def test_limb4_battery(gpu, p):
    # LIMB4 (16 MMAs, 7 accumulators, balanced base-256 digits, int64 fold): the seeded oracle
    # battery of test_random_battery over primes in (2^24, 2^31 - 1), plain and accumulating
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p % 100003)
    for t in range(8):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, 300))
        thr = (2, 8, 64, 16)[t % 4]
        a = orc.random_matrix(p, n, k, int(rng.integers(1 << 62)))
        plan = fs.make_syrk_plan(f, fs.RecursionPolicy(thr), mirror_output=(t == 5))
        want = orc.syrk_classical(p, a)
        if t % 2:
            alpha, beta = int(rng.integers(p)), int(rng.integers(p))
            c0 = orc.random_matrix(p, n, n, int(rng.integers(1 << 62)))
            c = c0.copy()
            fs.syrk_fast_acc(f, alpha, a, beta, c, plan)
            idx = np.tril_indices(n)
            exp = [(int(w) * alpha + int(x) * beta) % p for w, x in zip(want[idx], c0[idx])]
            assert np.array_equal(c[idx], np.array(exp, dtype=np.uint64)), (p, n, k, thr)
        else:
            c = fs.syrk_fast(f, a, plan)
            assert orc.lower_equal(c, want), (p, n, k, thr)


@pytest.mark.parametrize("p", LIMB4_PRIMES)
def test_limb4_extreme_values(gpu, p):
    # residues at the balanced-digit window edges and p - 1 through every limb
    fs = gpu
    f = fs.PrimeField(p)
    for val in (p - 1, p // 2, p // 2 + 1, 1, 0x80808080 % p, 0x7F7F7F7F % p):
        a = np.full((96, 160), val, dtype=np.uint64)
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(8)))
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, val)


@pytest.mark.parametrize("p", [998244353, 2147483629])
def test_limb4_syrkd_and_white_box(gpu, p):
    # LIMB4 through the syrkd column map and one level's S1..S4 / P1..P5 against the oracle
    fs = gpu
    f = fs.PrimeField(p)
    a = orc.random_matrix(p, 200, 150, 41)
    d = orc.random_nonzero(p, 150, 42)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(8))
    assert orc.lower_equal(fs.syrkd(f, a, d, plan), orc.syrkd(p, a, d, 8))
    for n, k in ((64, 48), (32, 32)):
        a = orc.random_matrix(p, n, k, 321)
        dev = fs.level_blocks(f, a)
        ref = orc.level_blocks(p, a)
        for key in ("S1", "S2", "S3", "S4", "P3", "P4"):
            assert np.array_equal(dev[key], ref[key]), (p, n, k, key)
        for key in ("P1", "P2", "P5"):
            assert orc.lower_equal(dev[key], ref[key]), (p, n, k, key)
