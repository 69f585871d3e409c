"""Host transfer format of the host entry points (host_io.cu), checked without a device:
the caller's rows are packed exactly as they go on the wire (B-bit groups of 32 residues, or
uint32) by the library's host worker pool and unpacked back.  The device half of the format
(unpack_kernel / pack_kernel) is covered by the GPU tests that go through the host entry
points (test_gpu_parity.py::test_host_io_*, test_triangular_host_transfers)."""
import numpy as np
import pytest


@pytest.mark.parametrize("bits", [8, 13, 16, 17, 23, 24, 32])
@pytest.mark.parametrize("lower,rows,cols", [(False, 1, 1), (False, 7, 33), (False, 333, 1001), (True, 1, 1),
                                             (True, 65, 65), (True, 1500, 1503), (False, 1100, 1000)])
def test_roundtrip_exact(fsyrk, bits, lower, rows, cols):
    rng = np.random.default_rng(bits * 1000 + rows)
    top = (1 << bits) if bits < 32 else (1 << 32)
    big = rng.integers(0, top, size=(rows, cols + 5), dtype=np.uint64)
    a = big[:, 2:2 + cols]  # strided rows
    out, raw, secs = fsyrk.hostio_roundtrip(a, lower, bits)
    mask = np.tril(np.ones((rows, cols), dtype=bool)) if lower else np.ones((rows, cols), dtype=bool)
    assert raw == 0
    assert np.array_equal(out[mask], a[mask])
    assert (out[~mask] == 0).all()
    assert secs[0] >= 0 and secs[1] >= 0


@pytest.mark.parametrize("bits", [17, 32])
def test_roundtrip_flags_oversize_values(fsyrk, bits):
    # a value that does not fit the transfer width marks its chunk for the unnarrowed copy
    # (1 Mi-element chunks of whole rows: 1100 x 1000 is two chunks)
    a = np.zeros((1100, 1000), dtype=np.uint64)
    a[1099, 999] = (1 << bits) + 5
    assert fsyrk.hostio_roundtrip(a, False, bits)[1] == 1
    a[0, 0] = 1 << 62
    assert fsyrk.hostio_roundtrip(a, False, bits)[1] == 2


def test_transfer_bits(fsyrk):
    assert fsyrk.transfer_bits(3) == 8
    assert fsyrk.transfer_bits(65521) == 16
    assert fsyrk.transfer_bits(65537) == 17
    assert fsyrk.transfer_bits(131071) == 17
    assert fsyrk.transfer_bits(2147483647) == 32


def test_roundtrip_in_forked_child(fsyrk):
    # the worker pool is per process: a child forked after the pool started builds its own
    import multiprocessing as mp
    a = np.arange(64 * 100, dtype=np.uint64).reshape(64, 100) % 65521
    fsyrk.hostio_roundtrip(a, False, 16)  # start the parent's pool
    ctx = mp.get_context("fork")
    q = ctx.Queue()

    def child(queue):
        out, raw, _ = fsyrk.hostio_roundtrip(a, False, 16)
        queue.put(bool(np.array_equal(out, a)) and raw == 0)

    proc = ctx.Process(target=child, args=(q,))
    proc.start()
    proc.join(60)
    assert proc.exitcode == 0 and q.get(timeout=5)


def test_roundtrip_from_several_threads(fsyrk):
    # the host worker pool serves one transfer at a time; concurrent callers queue up
    import threading
    rng = np.random.default_rng(5)
    mats = [rng.integers(0, 1 << 17, size=(700, 900), dtype=np.uint64) for _ in range(4)]
    ok = {}

    def work(t):
        good = True
        for _ in range(5):
            out, raw, _ = fsyrk.hostio_roundtrip(mats[t], False, 17)
            good &= bool(np.array_equal(out, mats[t])) and raw == 0
        ok[t] = good

    ths = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join(60)
    assert ok == {0: True, 1: True, 2: True, 3: True}
