"""Low-memory schedule (fsyrk_b200_set_workspace_limit) against the C oracle.

With a workspace limit below a plan's wide workspace, the top level's general products
P4, P3 are written into the scratch quadrant C12 of the caller's C -- the reference keeps its
S blocks and temporaries inside C the same way (fast_syrk.hpp:62-81, 96-98) -- and the root
post-addition reads them from there.  Low(C) must be bit-identical to the oracle for plain,
accumulating, syrkd and device-pointer calls; the schedule must actually be taken
(last_plan()["schedule"]) and report a smaller workspace; a limit below even the low-memory
workspace is refused.
"""
import numpy as np
import pytest

import oracle_py as orc

pytestmark = pytest.mark.gpu


@pytest.fixture
def limit(gpu):
    yield gpu.set_workspace_limit
    gpu.set_workspace_limit(0)
    gpu.set_low_memory(False)
    gpu.release_cache()


def _force_lowmem(fs, p, n, k, pol):
    wide = fs.workspace_bytes(p, n, k, pol)["arena"]
    lm = fs.workspace_bytes(p, n, k, pol, lowmem=True)["arena"]
    assert lm < wide
    fs.set_workspace_limit(wide - 1)
    return wide, lm


@pytest.mark.parametrize("p", [131071, 65537, 65521, 2147483647, 998244353, 11])
def test_lowmem_plain(gpu, limit, p):
    fs = gpu
    f = fs.PrimeField(p)
    for (n, k, thr) in ((256, 256, 64), (192, 160, 32), (512, 128, 2), (384, 200, 16)):
        pol = fs.RecursionPolicy(thr)
        _force_lowmem(fs, p, n, k, pol)
        a = orc.random_matrix(p, n, k, n + k)
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, pol))
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, n, k, thr)
        assert fs.last_plan()["schedule"] == "low-memory", (p, n, k)


@pytest.mark.parametrize("p", [131071, 65521, 2147483647])
def test_lowmem_accumulate_and_syrkd(gpu, limit, p):
    fs = gpu
    f = fs.PrimeField(p)
    rng = np.random.default_rng(p % 977)
    n, k = 256, 192
    pol = fs.RecursionPolicy(32)
    _force_lowmem(fs, p, n, k, pol)
    a = orc.random_matrix(p, n, k, 5)
    c0 = orc.random_matrix(p, n, n, 6)
    alpha, beta = int(rng.integers(1, p)), int(rng.integers(1, p))
    c = c0.copy()
    fs.syrk_fast_acc(f, alpha, a, beta, c, fs.make_syrk_plan(f, pol))
    assert orc.lower_equal(c, orc.syrk_classical(p, a, alpha, beta, c0))
    assert fs.last_plan()["schedule"] == "low-memory"
    # squares: no non-residue pairs left over, so k stays even and the top level a 2 x 2 level
    d = [int(x) * int(x) % p for x in rng.integers(1, p, size=k)]
    fs.set_low_memory(True)  # the syrkd plan's workspace differs (column map, residue input)
    c = c0.copy()
    fs.syrkd(f, a, d, fs.make_syrk_plan(f, pol), alpha=p - 1, beta=1, c=c)
    assert fs.last_plan()["schedule"] == "low-memory"
    x = orc.syrkd(p, a, d, 32)  # Low(A D A^T)
    want = (c0 + (np.uint64(p) - x) % np.uint64(p)) % np.uint64(p)
    assert orc.lower_equal(c, want)


def test_lowmem_device_pointers_and_limits(gpu, limit):
    torch = pytest.importorskip("torch")
    fs = gpu
    p, n, k = 131071, 512, 512
    pol = fs.RecursionPolicy(128)
    wide, lm = _force_lowmem(fs, p, n, k, pol)
    a = orc.random_matrix(p, n, k, 77)
    ad = torch.from_numpy(a.view(np.int64)).cuda()
    cd = torch.zeros((n, n), dtype=torch.int64, device="cuda")
    fs.syrk_dev(p, 1, ad.data_ptr(), n, k, k, 0, cd.data_ptr(), n, pol, False, 0)
    torch.cuda.synchronize()
    c = cd.cpu().numpy().view(np.uint64)
    assert orc.lower_equal(c, orc.syrk_classical(p, a))
    # an odd row stride cannot hold P4 | P3 pairs in C12: refused, not silently wrong
    cd2 = torch.zeros((n, n + 1), dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        fs.syrk_dev(p, 1, ad.data_ptr(), n, k, k, 0, cd2.data_ptr(), n + 1, pol, False, 0)
    # a limit below the low-memory workspace is refused
    fs.set_workspace_limit(lm - 1)
    fs.release_cache()
    with pytest.raises(ValueError):
        fs.syrk_dev(p, 1, ad.data_ptr(), n, k, k, 0, cd.data_ptr(), n, pol, False, 0)
