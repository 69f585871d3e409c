"""Device-path parity: the CUDA implementation, called through the C ABI,
against the reference's golden outputs and the pinned C oracle.

Bit-exact on every entry of Low(C) (integer arithmetic; no tolerance)."""
import os

import numpy as np
import pytest

import oracle_py as orc

pytestmark = pytest.mark.gpu

UNL = (1 << 64) - 1


def _policy(fs, case):
    return fs.RecursionPolicy(case["threshold"], UNL if case["levels"] is None else case["levels"])


def _blocks(fs, rows):
    bd = fs.BlockDiagonal()
    for two, d, beta, gamma in rows:
        bd.blocks.append(fs.BlockDiagonal.two_by_two(int(beta), int(gamma)) if two else fs.BlockDiagonal.scalar(int(d)))
    return bd


def test_golden_cases(gpu, golden):
    fs = gpu
    for case in golden["cases"]:
        f = fs.PrimeField(case["p"])
        plan = fs.make_syrk_plan(f, _policy(fs, case), mirror_output=case["mirror"])
        a = case["A"]
        if case["mode"] == "plain":
            c = fs.syrk_fast(f, a, plan)
        elif case["mode"] == "acc":
            c = case["C0"].copy()
            fs.syrk_fast_acc(f, case["alpha"], a, case["beta"], c, plan)
        elif case["mode"] in ("herk", "syrk2"):
            q = fs.QuadExtField(case["p"])
            if case["mode"] == "herk":
                c = fs.herk_fast(q, a, fs.make_herk_plan(q, _policy(fs, case)))
            else:
                c = fs.syrk_fast_fp2(q, a, fs.make_syrk_plan(f, _policy(fs, case)))
            for i in range(case["n"]):
                assert np.array_equal(c[i, :i + 1], case["C"][i, :i + 1]), (case["mode"], case["p"], case["n"], i)
            continue
        elif case["mode"] == "syrkbd":
            c = fs.syrkbd(f, a, _blocks(fs, case["D"]), plan)
        else:
            c = case["C0"].copy()
            fs.syrkd(f, a, case["D"], plan, alpha=case["p"] - 1, beta=1, c=c)
        assert orc.lower_equal(c, case["C"]), (case["mode"], case["p"], case["n"], case["k"])
        if case["mirror"]:
            assert np.array_equal(c, c.T)


def test_known_answers(gpu):
    fs = gpu
    # 2x2 over F_5 (test_fast_syrk.cpp:54-69): Low = [[0], [1, 0]]
    f = fs.PrimeField(5)
    a = np.array([[1, 2], [3, 4]], dtype=np.uint64)
    c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(2)))
    assert (c[0, 0], c[1, 0], c[1, 1]) == (0, 1, 0)
    # CLI round trip (cli_syrk_roundtrip.cmake:13-16, 37-40): mod 101
    f = fs.PrimeField(101)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy())
    c = fs.syrk_fast(f, a, plan)
    assert (c[0, 0], c[1, 0], c[1, 1]) == (5, 11, 25) and c[0, 1] == 0
    cm = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(), mirror_output=True))
    assert cm.tolist() == [[5, 11], [11, 25]]
    c0 = np.eye(2, dtype=np.uint64)
    fs.syrk_fast_acc(f, 2, a, 3, c0, plan)
    assert (c0[0, 0], c0[1, 0], c0[1, 1]) == (13, 22, 53)
    # syrkd examples (test_scaled_syrk.cpp:59-100)
    f7 = fs.PrimeField(7)
    p7 = fs.make_syrk_plan(f7, fs.RecursionPolicy(2))
    c = fs.syrkd(f7, np.eye(2, dtype=np.uint64), [3, 5], p7)
    assert (c[0, 0], c[1, 0], c[1, 1]) == (3, 0, 5)
    c = fs.syrkd(f7, np.ones((1, 1), dtype=np.uint64), [3], p7)
    assert c[0, 0] == 3


def test_degenerate(gpu):
    fs = gpu
    f = fs.PrimeField(131071)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(2))
    z = fs.syrk_fast(f, np.zeros((16, 16), dtype=np.uint64), plan)
    assert not np.tril(z).any()
    i = fs.syrk_fast(f, np.eye(16, dtype=np.uint64), plan)
    assert np.array_equal(np.tril(i), np.eye(16, dtype=np.uint64))
    # empty inputs
    assert fs.syrk_fast(f, np.zeros((0, 5), dtype=np.uint64), plan).shape == (0, 0)
    c = np.full((3, 3), 9, dtype=np.uint64)
    fs.syrk_fast_acc(f, 1, np.zeros((3, 0), dtype=np.uint64), 2, c, plan)
    assert np.array_equal(np.tril(c), np.tril(np.full((3, 3), 18, dtype=np.uint64)))
    # alpha = 0, beta = 1 leaves Low(C) unchanged; beta = 0 ignores C
    a = fs.random_matrix(f, 32, 32, 10)
    c0 = fs.random_matrix(f, 32, 32, 11)
    c = c0.copy()
    fs.syrk_fast_acc(f, 0, a, 1, c, plan)
    assert orc.lower_equal(c, c0)
    c = np.full((32, 32), 12345, dtype=np.uint64)
    fs.syrk_fast_acc(f, 7, a, 0, c, plan)
    assert orc.lower_equal(c, (orc.syrk_classical(131071, a) * np.uint64(7)) % np.uint64(131071))


@pytest.mark.parametrize("p", [5, 13, 131041, 2, 3, 11, 7, 131071, 65537, 65521, 2147483647])
def test_random_battery(gpu, p):
    # oracle battery (test_fast_syrk.cpp:71-98, acceptance.cpp:45-74), n, k <= 300
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p * 1009)
    for t in range(6):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, 300))
        thr = (2, 8, 64)[t % 3]
        a = orc.random_matrix(p, n, k, int(rng.integers(1 << 62)))
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(thr)))
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, n, k, thr)


def test_white_box_level(gpu):
    fs = gpu
    for p, n, k in ((131071, 8, 8), (131071, 64, 48), (65537, 32, 32), (11, 32, 10), (2147483647, 16, 16)):
        a = orc.random_matrix(p, n, k, 321)
        dev = fs.level_blocks(fs.PrimeField(p), a)
        ref = orc.level_blocks(p, a)
        assert dev["kw"] == ref["kw"]
        for key in ("S1", "S2", "S3", "S4", "P3", "P4"):
            assert np.array_equal(dev[key], ref[key]), (p, n, k, key)
        for key in ("P1", "P2", "P5"):
            assert orc.lower_equal(dev[key], ref[key]), (p, n, k, key)


@pytest.mark.parametrize("p", [65521, 65537, 131071, 2147483647])
def test_gemm_nt(gpu, p):
    fs = gpu
    f = fs.PrimeField(p)
    for (m, n, k) in ((1, 1, 1), (130, 97, 200), (256, 256, 256), (300, 129, 1000)):
        a = orc.random_matrix(p, m, k, 1)
        b = orc.random_matrix(p, n, k, 2)
        c = fs.gemm_nt(f, a, b)
        want = np.array([[orc.dot_mod(p, a[i], b[j]) for j in range(n)] for i in range(m)], dtype=np.uint64) \
            if m * n <= 4096 else None
        if want is None:
            full = np.vstack([a, b])
            s = orc.syrk_classical(p, full)
            want = s[m:, :m].T.copy()
        assert np.array_equal(c, want), (p, m, n, k)


def test_extreme_values(gpu):
    # all entries p-1 (largest magnitudes through every limb) and max-window residues
    fs = gpu
    for p in (65521, 65537, 131071, 2147483647):
        f = fs.PrimeField(p)
        for val in (p - 1, p // 2, p // 2 + 1, 1):
            a = np.full((96, 160), val, dtype=np.uint64)
            c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(8)))
            assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, val)


@pytest.mark.parametrize("p,k", [(2147483647, 8192), (131071, 32768), (65521, 32768), (65537, 16384)])
def test_accumulator_bounds_at_long_k(gpu, p, k):
    # largest digits everywhere at the inner dimensions the planner allows: the int32
    # accumulators and the fold must stay exact (schemes.cuh, modmm_k_limit)
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(k)
    for val in (p - 1, None):
        a = np.full((128, k), p - 1, dtype=np.uint64) if val else orc.random_matrix(p, 128, k, 5)
        b = np.full((96, k), p - 1, dtype=np.uint64) if val else orc.random_matrix(p, 96, k, 6)
        if val is None:
            a[:, ::3] = p - 1  # mix maximal and random digits
        c = fs.gemm_nt(f, a, b)
        full = orc.syrk_classical(p, np.vstack([a, b]))
        assert np.array_equal(c, full[128:, :128].T), (p, k)
    del rng


def test_mirror_and_strided_views(gpu):
    fs = gpu
    p = 131071
    f = fs.PrimeField(p)
    big = orc.random_matrix(p, 80, 100, 3)
    a = big[:, 10:74]  # strided view, lda = 100
    c_big = np.full((80, 90), 5, dtype=np.uint64)
    c = c_big[:, 3:83]
    fs.syrk_fast_into(f, a, c, fs.make_syrk_plan(f, fs.RecursionPolicy(4), mirror_output=True))
    want = orc.syrk_classical(p, np.ascontiguousarray(a))
    assert orc.lower_equal(np.ascontiguousarray(c), want)
    assert np.array_equal(c, c.T)
    assert (c_big[:, :3] == 5).all() and (c_big[:, 83:] == 5).all()
    # without mirroring the strict upper triangle is scratch (fast_syrk.hpp:271-273): the host
    # path clears it for beta = 0 and keeps the caller's values when C is read (beta != 0)
    c2 = np.full((80, 80), 77, dtype=np.uint64)
    fs.syrk_fast_into(f, a, c2, fs.make_syrk_plan(f, fs.RecursionPolicy(4)))
    assert (c2[np.triu_indices(80, 1)] == 0).all()
    c3 = np.full((80, 80), 77, dtype=np.uint64)
    fs.syrk_fast_acc(f, 1, a, 1, c3, fs.make_syrk_plan(f, fs.RecursionPolicy(4)))
    assert (c3[np.triu_indices(80, 1)] == 77).all()


def _random_blocks(rng, p, k):
    rows, dim = [], 0
    while dim < k:
        if rng.integers(3) == 0 or dim + 1 == k:
            rows.append((0, int(rng.integers(p)), 0, 0))
            dim += 1
        else:
            rows.append((1, 0, int(rng.integers(1, p)), 0))
            dim += 2
    return rows


@pytest.mark.parametrize("p", [3, 7, 13, 65521, 65537, 131071, 2147483647])
def test_syrkbd_battery(gpu, p):
    # scaled battery (acceptance.cpp:277-345): syrkbd against the dense A B A^T oracle, plain and in
    # the accumulating Schur form; odd / even non-residue counts, all-antidiagonal and all-scalar B
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p + 17)
    for t in range(8):
        n = int(rng.integers(1, 200))
        k = int(rng.integers(1, 160))
        rows = _random_blocks(rng, p, k)
        if t == 6 and k % 2 == 0:
            rows = [(1, 0, int(rng.integers(1, p)), 0) for _ in range(k // 2)]
        if t == 7:
            rows = [(0, int(rng.integers(p)), 0, 0) for _ in range(k)]
        a = orc.random_matrix(p, n, k, int(rng.integers(1 << 62)))
        thr = (2, 8, 64)[t % 3]
        plan = fs.make_syrk_plan(f, fs.RecursionPolicy(thr))
        want = orc.abat_classical(p, a, rows)
        c = fs.syrkbd(f, a, _blocks(fs, rows), plan)
        assert orc.lower_equal(c, want), (p, n, k, t)
        c0 = orc.random_matrix(p, n, n, 99)
        c = c0.copy()
        fs.syrkbd(f, a, _blocks(fs, rows), plan, alpha=p - 1, beta=1, c=c)
        idx = np.tril_indices(n)
        exp = c0.copy()
        exp[idx] = (c0[idx] + np.uint64(p) - want[idx]) % np.uint64(p)
        assert orc.lower_equal(c, exp), (p, n, k, t, "schur")


def test_syrkbd_examples_and_errors(gpu):
    fs = gpu
    # antidiagonal over F_7, A = I2, beta = 1 (test_scaled_syrk.cpp:151-161): Low = [[0], [1, 0]]
    f7 = fs.PrimeField(7)
    bd = fs.BlockDiagonal([fs.BlockDiagonal.two_by_two(1, 0)])
    c = fs.syrkbd(f7, np.eye(2, dtype=np.uint64), bd, fs.make_syrk_plan(f7, fs.RecursionPolicy(2)))
    assert (c[0, 0], c[1, 0], c[1, 1]) == (0, 1, 0)
    # scalar identity blocks reduce to plain syrk (:139-149)
    f13 = fs.PrimeField(13)
    a = fs.random_matrix(f13, 5, 5, 2)
    plan = fs.make_syrk_plan(f13, fs.RecursionPolicy(2))
    c = fs.syrkbd(f13, a, fs.BlockDiagonal([fs.BlockDiagonal.scalar(1)] * 5), plan)
    assert orc.lower_equal(c, fs.syrk_fast(f13, a, plan))
    # malformed blocks (:192-205): beta = 0, gamma != 0 in odd characteristic, dimension mismatch
    a2 = np.ones((2, 2), dtype=np.uint64)
    with pytest.raises(ValueError):
        fs.syrkbd(f7, a2, fs.BlockDiagonal([fs.BlockDiagonal.two_by_two(0, 0)]), plan)
    with pytest.raises(ValueError):
        fs.syrkbd(f7, a2, fs.BlockDiagonal([fs.BlockDiagonal.two_by_two(1, 1)]), plan)
    with pytest.raises(fs.DimensionError):
        fs.syrkbd(f7, a2, fs.BlockDiagonal([fs.BlockDiagonal.scalar(1)]), plan)


@pytest.mark.parametrize("p", [65521, 131071])
def test_split_k_child_alignment(gpu, p):
    # k > n splits k at k1 = (k/2) & ~1 (fast_syrk.hpp:143-150); k1 = 102 puts the second half at a
    # column offset that is not 16-byte aligned for residue rows while that child (k = 104) is
    # otherwise vector-shaped -- the prep must take its scalar path there
    fs = gpu
    f = fs.PrimeField(p)
    a = orc.random_matrix(p, 128, 206, 77)
    d = orc.random_nonzero(p, 206, 78)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(8))
    assert orc.lower_equal(fs.syrk_fast(f, a, plan), orc.syrk_classical(p, a))
    want = orc.syrkd(p, a, d, 8)
    assert orc.lower_equal(fs.syrkd(f, a, d, plan), want)


def _xfer_bytes(p, rows, cols, lower):
    """PCIe bytes host_io moves for a region (host_io.cu make_chunks / transfer_bits): row-aligned
    chunks of <= 2^20 elements, each a stream of B-bit groups of 32 residues (B = bit length of
    p - 1, at least 8, when <= 24) or of uint32."""
    b = max(8, (p - 1).bit_length())
    width = (lambda i: i + 1) if lower else (lambda i: cols)
    cap = max(1 << 20, rows if lower else cols)
    total, r0 = 0, 0
    while r0 < rows:
        r1, ln = r0, 0
        while r1 < rows and (ln == 0 or ln + width(r1) <= cap):
            ln += width(r1)
            r1 += 1
        total += (ln + 31) // 32 * b * 4 if b <= 24 else ln * 4
        r0 = r1
    return total


def test_triangular_host_transfers(gpu):
    # only Low(C) crosses PCIe: results stay exact across chunk edges, the byte count matches,
    # beta = 0 clears the diagonal blocks' strict upper parts, beta != 0
    # leaves the caller's strict upper triangle as it was
    fs = gpu
    p, n, k = 131071, 600, 200
    f = fs.PrimeField(p)
    a = orc.random_matrix(p, n, k, 5)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(16))
    want = orc.syrk_classical(p, a)
    c = np.full((n, n), 7, dtype=np.uint64)
    fs.syrk_fast_into(f, a, c, plan)
    assert orc.lower_equal(c, want)
    blocks = [(r0, min(n, r0 + 256)) for r0 in range(0, n, 256)]
    # residues cross PCIe bit-packed (17 bits here; packed / unpacked by host threads, host_io.h)
    assert fs.last_transfer_bytes() == (_xfer_bytes(p, n, k, False), _xfer_bytes(p, n, n, True))
    for r0, r1 in blocks:
        blk = c[r0:r1, r0:r1]
        assert (blk[np.triu_indices(r1 - r0, 1)] == 0).all()
    assert (c[:256, 256:] == 7).all()
    c0 = orc.random_matrix(p, n, n, 6)
    c = c0.copy()
    fs.syrk_fast_acc(f, 3, a, 5, c, plan)
    idx = np.tril_indices(n)
    exp = c0.copy()
    exp[idx] = (want[idx] * np.uint64(3) + c0[idx] * np.uint64(5)) % np.uint64(p)
    assert orc.lower_equal(c, exp)
    assert np.array_equal(c[np.triu_indices(n, 1)], c0[np.triu_indices(n, 1)])


def _pinned(shape):
    torch = pytest.importorskip("torch")
    t = torch.empty(shape, dtype=torch.int64, pin_memory=True)
    return t.numpy().view(np.uint64)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("p", [2147483647, 131071, 65521])
def test_host_io_chunked_paths(gpu, pinned, p):
    # host_io: several 2 Mi-element chunks each way (A narrowed in host threads, Low(C) widened),
    # strided caller views, and with pinned C the accumulate duplex path (raw row blocks of C_in
    # and C out at the same time); pageable C takes the narrowed path for C_in too
    fs = gpu
    n, k = 2300, 1500
    f = fs.PrimeField(p)
    big = orc.random_matrix(p, n, k + 7, 11)
    a = big[:, 3:3 + k]
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(256, 2))
    want = orc.syrk_classical(p, np.ascontiguousarray(a))
    cbig = _pinned((n, n + 5)) if pinned else np.empty((n, n + 5), dtype=np.uint64)
    cbig[:] = 9
    c = cbig[:, 2:2 + n]
    fs.syrk_fast_into(f, a, c, plan)
    assert orc.lower_equal(np.ascontiguousarray(c), want)
    assert (cbig[:, :2] == 9).all() and (cbig[:, 2 + n:] == 9).all()
    h2d, d2h = fs.last_transfer_bytes()  # pinned C: a share of the rows also moves unnarrowed
    want_a, want_c = _xfer_bytes(p, n, k, False), _xfer_bytes(p, n, n, True)
    assert h2d == want_a and (d2h >= want_c if pinned else d2h == want_c)
    c0 = orc.random_matrix(p, n, n, 12)
    c[:] = c0
    alpha, beta = 123456789, 987654321
    fs.syrk_fast_acc(f, alpha, a, beta, c, plan)
    idx = np.tril_indices(n)
    exp = c0.copy()
    exp[idx] = np.array([(int(w) * alpha + int(x) * beta) % p for w, x in zip(want[idx], c0[idx])], dtype=np.uint64)
    assert np.array_equal(np.ascontiguousarray(c)[idx], exp[idx])
    assert np.array_equal(np.ascontiguousarray(c)[np.triu_indices(n, 1)], c0[np.triu_indices(n, 1)])
    assert (cbig[:, :2] == 9).all() and (cbig[:, 2 + n:] == 9).all()
    h2d, d2h = fs.last_transfer_bytes()
    assert h2d >= want_a and d2h >= want_c


def test_host_io_noncanonical_inputs(gpu):
    # values >= 2^32 cannot be narrowed: their chunk crosses PCIe as uint64 and the device
    # reduces them (the reference's PrimeField treats stored words as residues mod p only
    # after reduction; the device path reduces any uint64)
    fs = gpu
    p, n, k = 131071, 300, 200
    f = fs.PrimeField(p)
    a = orc.random_matrix(p, n, k, 21)
    big = a.copy()
    big[5, 7] += np.uint64(p) * np.uint64(1 << 40)
    big[250, 3] += np.uint64(p) * np.uint64(3)
    a[100, 100] = 0
    big[100, 100] = p
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(32))
    want = orc.syrk_classical(p, a)
    fits = a.copy()
    fits[100, 100] = p  # fits the 17-bit transfer width: crosses packed, the device reduces it
    assert orc.lower_equal(fs.syrk_fast(f, fits, plan), want)
    assert orc.lower_equal(fs.syrk_fast(f, big, plan), want)
    c0 = orc.random_matrix(p, n, n, 22)
    c = c0.copy()
    c[10, 2] += np.uint64(p) * np.uint64(1 << 33)
    fs.syrk_fast_acc(f, 1, a, 1, c, plan)
    idx = np.tril_indices(n)
    assert np.array_equal(c[idx], (want[idx] + c0[idx]) % np.uint64(p))


@pytest.mark.parametrize("p", [3, 7, 13, 65521, 131071, 2147483647])
def test_fp2_herk_and_syrk_battery(gpu, p):
    # herk_fast / syrk_fast over F_{p^2} (fast_syrk.hpp:305-320; verify_herk_battery, fsyrk.cpp)
    # against the classical conjugate product; mirror gives conj(C)^T / C^T above the diagonal
    fs = gpu
    q = fs.QuadExtField(p)
    rng = np.random.default_rng(p + 3)
    for t in range(4):
        n = int(rng.integers(1, 150))
        k = int(rng.integers(1, 120))
        a = orc.random_matrix(p, n, 2 * k, int(rng.integers(1 << 62))).reshape(n, k, 2)
        pol = fs.RecursionPolicy((2, 8, 64, 16)[t])
        want_h = orc.fp2_syrk_classical(p, a, True)
        want_s = orc.fp2_syrk_classical(p, a, False)
        c = fs.herk_fast(q, a, fs.make_herk_plan(q, pol, mirror_output=True))
        cs = fs.syrk_fast_fp2(q, a, fs.make_syrk_plan(q.base, pol, mirror_output=True))
        for i in range(n):
            assert np.array_equal(c[i, :i + 1], want_h[i, :i + 1]), (p, n, k, i)
            assert np.array_equal(cs[i, :i + 1], want_s[i, :i + 1]), (p, n, k, i)
        iu = np.triu_indices(n, 1)
        assert np.array_equal(c[iu][:, 0], c.transpose(1, 0, 2)[iu][:, 0])                # Hermitian
        assert np.array_equal(c[iu][:, 1], (np.uint64(p) - c.transpose(1, 0, 2)[iu][:, 1]) % np.uint64(p))
        assert np.array_equal(cs[iu], cs.transpose(1, 0, 2)[iu])                           # symmetric
    with pytest.raises(ValueError):
        fs.herk_fast(q, np.zeros((2, 2, 2), np.uint64), fs.make_syrk_plan(q.base))       # not a herk plan


@pytest.mark.parametrize("p", [65521, 131071, 2147483647, 13])
def test_winograd_general_product(gpu, p):
    # Strassen-Winograd levels over the tensor-core product (winograd.hpp:118-169, test_winograd.cpp):
    # exact, so bit-identical to the direct product for every depth, odd sizes stopping the recursion
    fs = gpu
    f = fs.PrimeField(p)
    for (m, n, k, thr, lev) in ((64, 64, 64, 2, 1), (256, 128, 192, 16, 2), (96, 160, 64, 8, 3),
                                (130, 98, 70, 2, 4), (512, 512, 512, 64, 2), (33, 40, 50, 2, 3)):
        a = orc.random_matrix(p, m, k, m + k)
        b = orc.random_matrix(p, n, k, n + 3 * k)
        c = fs.gemm_winograd_nt(f, a, b, fs.RecursionPolicy(thr, lev))
        assert np.array_equal(c, fs.gemm_nt(f, a, b)), (p, m, n, k, lev)
    a = np.full((128, 128), p - 1, dtype=np.uint64)  # extreme residues through every level
    c = fs.gemm_winograd_nt(f, a, a, fs.RecursionPolicy(8, 3))
    assert np.array_equal(c, fs.gemm_nt(f, a, a))


@pytest.mark.parametrize("p", [131071, 65521, 65537, 2147483647])
def test_root_post_overlapped_with_products(gpu, p):
    # FSYRK_B200_POST_ROUNDS (off by default, read at first plan creation: this test runs in
    # its own process): one-level plans with h >= 2048 run the root post-addition as the
    # product kernel's programmatic dependent, pair by pair as the product rounds complete
    # (driver.cu Plan::nrounds); exact against the oracle, accumulating with alpha, beta
    import subprocess
    import sys
    if os.environ.get("FSYRK_B200_POST_ROUNDS") is None:
        env = dict(os.environ, FSYRK_B200_POST_ROUNDS="8", FSYRK_B200_ROUND_CTAS="120")
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            f"{__file__}::test_root_post_overlapped_with_products[{p}]"],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
        return
    fs = gpu
    f = fs.PrimeField(p)
    n, k = 4096, 96
    a = orc.random_matrix(p, n, k, 31)
    c0 = orc.random_matrix(p, n, n, 32)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(2, 1))
    alpha, beta = 12345 % p, 54321 % p
    c = c0.copy()
    fs.syrk_fast_acc(f, alpha, a, beta, c, plan)
    assert fs.last_plan()["post_rounds"] > 1
    want = orc.syrk_classical(p, a)
    idx = np.tril_indices(n)
    exp = (want[idx] * np.uint64(alpha) % np.uint64(p) + c0[idx] * np.uint64(beta) % np.uint64(p)) % np.uint64(p)
    assert np.array_equal(c[idx], exp)
    c2 = fs.syrk_fast(f, a, plan)
    assert orc.lower_equal(c2, want)


@pytest.mark.slow
@pytest.mark.parametrize("p", [5, 13, 131041, 3, 7, 11, 131071, 65521, 65537, 2147483647])
def test_acceptance_battery(gpu, p):
    # the reference's main parity gate at its own scale (acceptance.cpp:45-74): 500 seeded
    # cases per prime, n, k <= 256, thresholds {2, 8, 64}; every third case accumulates with
    # random alpha, beta (test_fast_syrk.cpp:312-375) and every fifth mirrors.  The reference's
    # seven primes plus the BASELINE primes of the other digit schemes (LIMB2, LIMB3, M31).
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p * 7919 + 1)
    for t in range(500):
        n = int(rng.integers(1, 257))
        k = int(rng.integers(1, 257))
        thr = (2, 8, 64)[t % 3]
        a = orc.random_matrix(p, n, k, int(rng.integers(1 << 62)))
        plan = fs.make_syrk_plan(f, fs.RecursionPolicy(thr), mirror_output=(t % 5 == 4))
        want = orc.syrk_classical(p, a)
        if t % 3 == 1:
            alpha, beta = int(rng.integers(p)), int(rng.integers(p))
            c0 = orc.random_matrix(p, n, n, int(rng.integers(1 << 62)))
            c = c0.copy()
            fs.syrk_fast_acc(f, alpha, a, beta, c, plan)
            idx = np.tril_indices(n)
            exp = (want[idx] * np.uint64(alpha) % np.uint64(p) + c0[idx] * np.uint64(beta) % np.uint64(p)) % np.uint64(p)
            assert np.array_equal(c[idx], exp), (p, n, k, thr, t)
        else:
            c = fs.syrk_fast(f, a, plan)
            assert orc.lower_equal(c, want), (p, n, k, thr, t)
            if t % 5 == 4:
                assert np.array_equal(c, c.T), (p, n, k, t)
        if t % 100 == 99:
            fs.release_cache()
    fs.release_cache()


def test_host_entry_rejects_device_memory(gpu):
    # the host entry points stage through host threads: device pointers are refused (EINVAL),
    # not dereferenced on the host
    torch = pytest.importorskip("torch")
    import ctypes
    fs = gpu
    lib = fs.lib()
    a = torch.zeros((64, 32), dtype=torch.int64, device="cuda")
    c = np.zeros((64, 64), dtype=np.uint64)
    pol = fs.RecursionPolicy(8)._c()
    u64p = ctypes.POINTER(ctypes.c_uint64)
    st = lib.fsyrk_b200_syrk_fast_into(131071, ctypes.cast(a.data_ptr(), u64p), 64, 32, 32,
                                       c.ctypes.data_as(u64p), 64, pol, 0, None)
    assert st == 2 and b"device memory" in lib.fsyrk_b200_last_error()


@pytest.mark.parametrize("p", [131071, 2147483647])
def test_upload_download_staging(gpu, p):
    # fsyrk_b200_upload / _download (the staging path of the host entry points, exposed for
    # device-resident callers such as rank 0 of a multi-GPU call): exact round trips, Low only
    torch = pytest.importorskip("torch")
    fs = gpu
    n, k = 1500, 1100
    a = orc.random_matrix(p, n, k, 41)
    a_dev = torch.zeros((n, k + 3), dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    fs.upload(p, a, a_dev.data_ptr(), k + 3, stream=s)
    torch.cuda.synchronize()
    assert np.array_equal(a_dev[:, :k].cpu().numpy().view(np.uint64), a)
    c = orc.random_matrix(p, n, n, 42)
    c_dev = torch.from_numpy(c.view(np.int64)).cuda()
    out = np.full((n, n), 7, dtype=np.uint64)
    fs.download(p, c_dev.data_ptr(), n, out, lower=True, stream=s)
    idx = np.tril_indices(n)
    assert np.array_equal(out[idx], c[idx]) and (out[np.triu_indices(n, 1)] == 7).all()
    up = fs.last_transfer_bytes()[1]
    assert 0 < up < n * (n + 1) // 2 * 8


def test_concurrent_host_calls(gpu):
    # host entry points called from several host threads at once (the staging path, plan cache
    # and worker pool are shared): every result exact
    import threading
    fs = gpu
    results = {}

    def work(tid):
        p = (131071, 65521, 2147483647, 65537)[tid % 4]
        f = fs.PrimeField(p)
        ok = True
        for it in range(6):
            n, k = 200 + 37 * tid + it, 150 + 11 * it
            a = orc.random_matrix(p, n, k, 1000 * tid + it)
            plan = fs.make_syrk_plan(f, fs.RecursionPolicy(16))
            if it % 2:
                c0 = orc.random_matrix(p, n, n, 7 + it)
                c = c0.copy()
                fs.syrk_fast_acc(f, 2, a, 3, c, plan)
                want = orc.syrk_classical(p, a)
                idx = np.tril_indices(n)
                ok &= bool(np.array_equal(c[idx], (want[idx] * np.uint64(2) % np.uint64(p)
                                                   + c0[idx] * np.uint64(3) % np.uint64(p)) % np.uint64(p)))
            else:
                ok &= orc.lower_equal(fs.syrk_fast(f, a, plan), orc.syrk_classical(p, a))
        results[tid] = ok

    threads = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(300)
    assert len(results) == 6 and all(results.values()), results


def test_concurrent_device_calls_share_a_plan(gpu):
    # device entry point from two host threads on two streams with the same shape: the calls
    # share one cached plan (arena), ordered by the plan's completion event; results exact
    import threading
    torch = pytest.importorskip("torch")
    fs = gpu
    p, n, k = 131071, 512, 384
    pol = fs.RecursionPolicy(64)
    inputs = [orc.random_matrix(p, n, k, 60 + t) for t in range(2)]
    wants = [orc.syrk_classical(p, a) for a in inputs]
    results = {}

    def work(t):
        stream = torch.cuda.Stream()
        a_dev = torch.from_numpy(inputs[t].view(np.int64)).cuda()
        ok = True
        with torch.cuda.stream(stream):
            for it in range(20):
                c_dev = torch.zeros((n, n), dtype=torch.int64, device="cuda")
                fs.syrk_dev(p, 1, a_dev.data_ptr(), n, k, k, 0, c_dev.data_ptr(), n, pol, False, stream.cuda_stream)
                stream.synchronize()
                ok &= orc.lower_equal(c_dev.cpu().numpy().view(np.uint64), wants[t])
        results[t] = ok

    threads = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(300)
    assert results == {0: True, 1: True}
