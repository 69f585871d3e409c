"""Multi-GPU partition of the top level.

CPU: the block-pair ownership is complete, disjoint and balanced, and the
multi-rank composition used by bench.py (disjoint shares summed over ranks,
max-over-ranks timing) is exercised with world_size 2 over gloo.
GPU: every rank's share computed on one device (ranks are independent: no rank
waits on another) reassembles bit-exactly into the single-GPU result."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_py as orc

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
def owner_mask(n, owners, rank, BLOCK):
    """Entries of Low(C) written by `rank` (C11 / C22 lower blocks, C21 by unordered pair)."""
    h = n // 2
    i, j = np.tril_indices(n)
    own = np.zeros(n * n, dtype=bool).reshape(n, n)
    top = i < h
    bi = np.where(top, i, i - h) // BLOCK
    bj = np.where(j < h, j, j - h) // BLOCK
    hi, lo = np.maximum(bi, bj), np.minimum(bi, bj)
    own[i, j] = owners[hi, lo] == rank
    return own


@pytest.mark.parametrize("p", [131071, 2147483647, 65521, 65537])
@pytest.mark.parametrize("h,nranks", [(2048, 2), (2048, 8), (8192, 8), (16384, 4), (500, 3), (384, 5)])
def test_partition_owners_complete_and_balanced(fsyrk, p, h, nranks):
    own, BLOCK = fsyrk.partition_owners(p, h, nranks)
    assert BLOCK % 128 == 0 and BLOCK % 32 == 0
    nb = (h + BLOCK - 1) // BLOCK
    assert own.shape == (nb, nb)
    lower = own[np.tril_indices(nb)]
    assert (lower >= 0).all() and (lower < nranks).all()
    assert (own[np.triu_indices(nb, 1)] == -1).all()
    rows = [min(BLOCK, h - b * BLOCK) for b in range(nb)]
    # per-rank work: its block pairs' products plus the pre-additions of every block they touch
    # (one block ~ one block pair of products, the planner's cost model)
    load = np.zeros(nranks)
    touched = [set() for _ in range(nranks)]
    for bi in range(nb):
        for bj in range(bi + 1):
            r = own[bi, bj]
            load[r] += rows[bi] * rows[bj] * (0.5 if bi == bj else 1.0)
            touched[r] |= {bi, bj}
    for r in range(nranks):
        load[r] += sum(rows[b] * BLOCK for b in touched[r])
    if nb * (nb + 1) // 2 >= 4 * nranks:
        assert load.max() / load.mean() < 1.2


def _gloo_worker(rank, world, port, n, p, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_py as o
    import paper_2001_04109_b200 as fs
    import bench
    a = o.random_matrix(p, n, n, 42)
    full = o.syrk_classical(p, a)
    owners, blk = fs.partition_owners(p, n // 2, world)
    mask = owner_mask(n, owners, rank, blk)
    share = np.where(mask, full, 0).astype(np.int64)  # what this rank's device C holds (beta = 0)
    t = torch.from_numpy(share)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)           # bench.py's gather of disjoint shares
    ms = bench.max_over_ranks(float(rank + 1), world)  # bench.py's timing reduction
    ok = np.array_equal(np.tril(t.numpy().astype(np.uint64)), np.tril(full)) and ms == float(world)
    result_q.put((rank, ok, int(mask.sum())))
    dist.destroy_process_group()


def test_two_rank_composition_over_gloo(fsyrk):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    n, p, world = 1536, 131071, 2
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert sum(c for _, _, c in res) == n * (n + 1) // 2  # every lower entry owned exactly once


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("mode", ["plain", "acc", "schur"])
def test_partition_shares_reassemble(gpu, nranks, mode):
    fs = gpu
    p, n, k = 131071, 1536, 1024
    f = fs.PrimeField(p)
    a = fs.random_matrix(f, n, k, 7)
    pol = fs.RecursionPolicy(2, 1)
    dev = torch.device("cuda")
    a_d = torch.from_numpy(a.view(np.int64)).to(dev)
    c0 = fs.random_matrix(f, n, n, 8) if mode != "plain" else np.zeros((n, n), np.uint64)
    alpha, beta, d = (1, 0, None) if mode == "plain" else (5, 7, None) if mode == "acc" else (p - 1, 1, None)
    if mode == "schur":
        d = orc.random_nonzero(p, k, 9)
    ref_d = torch.from_numpy(c0.view(np.int64).copy()).to(dev)
    fs.syrk_dev(p, alpha, a_d.data_ptr(), n, k, k, beta, ref_d.data_ptr(), n, pol, False, 0, d=d)
    c_d = torch.from_numpy(c0.view(np.int64).copy()).to(dev)
    for r in range(nranks):
        fs.syrk_part_dev(p, alpha, a_d.data_ptr(), n, k, k, beta, c_d.data_ptr(), n, pol, r, nranks, 0, d=d)
    torch.cuda.synchronize()
    got = c_d.cpu().numpy().view(np.uint64)
    want = ref_d.cpu().numpy().view(np.uint64)
    assert orc.lower_equal(got, want)
    # and each share writes only what its rank owns
    owners, blk = fs.partition_owners(p, n // 2, nranks)
    c1 = torch.zeros((n, n), dtype=torch.int64, device=dev)
    fs.syrk_part_dev(p, 1, a_d.data_ptr(), n, k, k, 0, c1.data_ptr(), n, pol, 1, nranks, 0)
    torch.cuda.synchronize()
    written = np.tril(c1.cpu().numpy()) != 0
    assert not (written & ~owner_mask(n, owners, 1, blk)).any()
