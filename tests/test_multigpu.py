"""Multi-GPU partition of the top level.

CPU: the block-pair ownership is complete, disjoint and balanced; the library's share tile
pairs cover Low(C) exactly once; and the data flow of the library's multi-GPU call
(fsyrk_b200_syrk_mgpu_rank: broadcast A, per-rank shares in the packed uint32 layout for the
library's tile pairs, gather to rank 0) runs with world_size 2 over gloo.
GPU: every rank's share computed on one device (ranks are independent: no rank
waits on another) reassembles bit-exactly into the single-GPU result, and the library's
multi-GPU entry point (loopback ranks on one device; a 1-rank NCCL communicator) matches
the oracle."""
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


def share_entries(pairs, h):
    """(slot, r, col) -> (row, col) of C for a share in the library's layout
    (include/fsyrk_b200.h fsyrk_b200_share_pairs): per pair (I, J), slots C11(I,J), C21(I,J),
    C22(I,J), C21(J,I) of 32 x 32 words; entries outside Low(C) or beyond h are unused."""
    idx_pos, idx_rc = [], []
    r, cl = np.meshgrid(np.arange(32), np.arange(32), indexing="ij")
    for q, (I, J) in enumerate(pairs):
        for t in range(4):
            if t == 3 and I == J:
                continue
            bi, bj = (J, I) if t == 3 else (I, J)
            li, lj = bi * 32 + r, bj * 32 + cl
            ok = (li < h) & (lj < h)
            if t in (0, 2) and I == J:
                ok &= cl <= r
            gi = li + (0 if t == 0 else h)
            gj = lj + (h if t == 2 else 0)
            pos = (q * 4 + t) * 1024 + r * 32 + cl
            idx_pos.append(pos[ok])
            idx_rc.append((gi[ok], gj[ok]))
    if not idx_pos:
        return np.zeros(0, np.int64), (np.zeros(0, np.int64), np.zeros(0, np.int64))
    return (np.concatenate(idx_pos), (np.concatenate([x[0] for x in idx_rc]), np.concatenate([x[1] for x in idx_rc])))


def _gloo_worker(rank, world, port, n, p, result_q):
    # the multi-GPU data flow of fsyrk_b200_syrk_mgpu_rank with gloo standing in for NCCL:
    # broadcast A (uint32 residues), each rank's share of Low(C) in the library's packed layout
    # for the tile pairs the library assigns it, gathered to rank 0 and unpacked
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_py as o
    import paper_2001_04109_b200 as fs
    import bench
    h = n // 2
    a32 = torch.zeros((n, n), dtype=torch.int32)
    if rank == 0:
        a32 = torch.from_numpy(o.random_matrix(p, n, n, 42).astype(np.int32))
    dist.broadcast(a32, src=0)
    a = a32.numpy().astype(np.uint64)
    full = o.syrk_classical(p, a)              # what every rank's device C would hold on its tiles
    pairs = [fs.share_pairs(p, h, r, world) for r in range(world)]
    pos, (gi, gj) = share_entries(pairs[rank], h)
    share = np.zeros(len(pairs[rank]) * 4096, dtype=np.int32)
    share[pos] = full[gi, gj].astype(np.int32)
    t = torch.from_numpy(share)
    if rank == 0:
        got = np.zeros((n, n), dtype=np.uint64)
        covered = np.zeros((n, n), dtype=np.int32)
        for r in range(world):
            buf = t if r == 0 else torch.zeros(len(pairs[r]) * 4096, dtype=torch.int32)
            if r:
                dist.recv(buf, src=r)
            pr, (ri, rj) = share_entries(pairs[r], h)
            got[ri, rj] = buf.numpy()[pr].astype(np.uint64)
            np.add.at(covered, (ri, rj), 1)
        ok = orc_lower_equal(got, full) and (covered[np.tril_indices(n)] == 1).all() and \
            not covered[np.triu_indices(n, 1)].any()
    else:
        dist.send(t, dst=0)
        ok = True
    ms = bench.max_over_ranks(float(rank + 1), world)  # bench.py's timing reduction
    result_q.put((rank, bool(ok) and ms == float(world), int(len(pos))))
    dist.destroy_process_group()


def orc_lower_equal(x, y):
    i = np.tril_indices(x.shape[0])
    return np.array_equal(x[i], y[i])


def test_share_pairs_partition_every_tile_once(fsyrk):
    # the owned tile pairs of all ranks cover the 32 x 32 tile pairs of the quadrants exactly once
    # and agree with partition_owners' block-pair owners
    for p, h, world in ((131071, 2048, 3), (2147483647, 1000, 4), (65521, 4096, 8)):
        own, blk = fsyrk.partition_owners(p, h, world)
        T = (h + 31) // 32
        seen = np.zeros((T, T), dtype=np.int32)
        for r in range(world):
            for I, J in fsyrk.share_pairs(p, h, r, world):
                assert I >= J and own[I * 32 // blk, J * 32 // blk] == r
                seen[I, J] += 1
        assert (seen[np.tril_indices(T)] == 1).all() and not seen[np.triu_indices(T, 1)].any()


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


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("mode", ["plain", "acc", "schur", "mirror"])
def test_syrk_mgpu_entry(gpu, devices, mode):
    # fsyrk_b200_syrk_mgpu: one GPU on this box, so >1 ranks are loopback ranks on device 0
    # (same partition, share packing, scatter of C_in and gather as over NCCL; the exchange is
    # device copies) -- bit-exact against the oracle
    fs = gpu
    p, n, k = 131071, 1600, 640
    f = fs.PrimeField(p)
    a = orc.random_matrix(p, n, k, 71)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(2, 1), mirror_output=(mode == "mirror"))
    want = orc.syrk_classical(p, a)
    c0 = orc.random_matrix(p, n, n, 72)
    c = c0.copy()
    idx = np.tril_indices(n)
    if mode in ("plain", "mirror"):
        fs.syrk_mgpu(f, a, c, plan, devices)
        assert orc.lower_equal(c, want)
        if mode == "mirror":
            assert np.array_equal(c, c.T)
    elif mode == "acc":
        fs.syrk_mgpu(f, a, c, plan, devices, alpha=5, beta=7)
        assert np.array_equal(c[idx], (want[idx] * np.uint64(5) + c0[idx] * np.uint64(7)) % np.uint64(p))
        assert np.array_equal(c[np.triu_indices(n, 1)], c0[np.triu_indices(n, 1)])
    else:
        d = orc.random_nonzero(p, k, 73)
        fs.syrk_mgpu(f, a, c, plan, devices, alpha=p - 1, beta=1, d=d)
        sd = orc.syrkd(p, a, d, 2)
        assert np.array_equal(c[idx], (c0[idx] + np.uint64(p) - sd[idx]) % np.uint64(p))


@pytest.mark.gpu
def test_syrk_mgpu_unpartitionable_and_odd_shapes(gpu):
    # shapes whose top level does not recurse (odd n) run on the first device alone; k = 0
    fs = gpu
    p = 2147483647
    f = fs.PrimeField(p)
    plan = fs.make_syrk_plan(f, fs.RecursionPolicy(2, 1))
    for n, k in ((301, 200), (256, 0), (640, 700)):
        a = orc.random_matrix(p, n, k, 74) if k else np.zeros((n, 0), np.uint64)
        c = np.full((n, n), 3, dtype=np.uint64)
        fs.syrk_mgpu(f, a, c, plan, [0, 0])
        assert orc.lower_equal(c, orc.syrk_classical(p, a) if k else np.zeros((n, n), np.uint64)), (n, k)


@pytest.mark.gpu
def test_communicator_single_rank(gpu):
    # the multi-process entry with a real NCCL communicator of one rank (the box has one GPU)
    fs = gpu
    p, n, k = 65521, 700, 500
    f = fs.PrimeField(p)
    comm = fs.Communicator(fs.nccl_unique_id(), 0, 1)
    try:
        a = orc.random_matrix(p, n, k, 75)
        c = np.zeros((n, n), dtype=np.uint64)
        comm.syrk(f, a, c, n, k, fs.make_syrk_plan(f, fs.RecursionPolicy(8)))
        assert orc.lower_equal(c, orc.syrk_classical(p, a))
    finally:
        comm.close()


def test_bench_gpus_flag_self_launches_torchrun(monkeypatch):
    # `bench.py --gpus N` without WORLD_SIZE starts N ranks itself (one process per GPU) with
    # torchrun on 127.0.0.1 and NCCL_DEBUG=INFO, instead of silently running one rank
    sys.path.insert(0, REPO)
    import bench
    seen = {}

    class _Done:
        returncode = 0

    def fake_run(cmd, env=None, **kw):
        seen["cmd"], seen["env"] = cmd, env
        return _Done()

    monkeypatch.setattr(torch.cuda, "device_count", lambda: 8)
    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=2" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
    assert cmd[-6:] == ["--gpus", "2", "--steps", "3", "--warmup", "3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
    # fewer visible devices than requested: refused, not a one-rank run
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 1)
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 2
