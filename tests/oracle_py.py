"""ctypes wrapper of the C oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: the checker for the device path.  Never imported
by the product package.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_SO = os.path.join(REPO, "oracle", "_build", "liboracle.so")
_u64p = ctypes.POINTER(ctypes.c_uint64)
_sz = ctypes.c_size_t
_u64 = ctypes.c_uint64
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            subprocess.run(["make", "-C", os.path.join(REPO, "oracle"), os.path.join(REPO, "oracle", "_build",
                                                                                     "liboracle.so")], check=True)
        L = ctypes.CDLL(_SO)
        L.orc_mt64_stream.argtypes = [_u64, _sz, _u64p]
        L.orc_random_matrix.argtypes = [_u64, _sz, _sz, _u64, _u64p]
        L.orc_random_nonzero.argtypes = [_u64, _sz, _u64, _u64p]
        L.orc_alpha_beta.argtypes = [_u64, _u64, _u64p, _u64p]
        L.orc_is_prime.argtypes = [_u64]
        L.orc_legendre.argtypes = [_u64, _u64]
        L.orc_sqrt.argtypes = [_u64, _u64]
        L.orc_sqrt.restype = _u64
        L.orc_lqnr.argtypes = [_u64]
        L.orc_lqnr.restype = _u64
        L.orc_skew.argtypes = [_u64, ctypes.POINTER(ctypes.c_int), _u64p, _u64p, ctypes.POINTER(ctypes.c_int)]
        L.orc_nrsyf.argtypes = [_u64, _u64, _u64, _u64p]
        L.orc_syrk_classical.argtypes = [_u64, _u64, _u64p, _sz, _sz, _sz, _u64, _u64p, _sz]
        L.orc_syrk_fast.argtypes = [_u64, _u64p, _sz, _sz, _sz, _u64p, _sz, _sz, _sz]
        L.orc_syrk_fast_acc.argtypes = [_u64, _u64, _u64p, _sz, _sz, _sz, _u64, _u64p, _sz, _sz, _sz]
        L.orc_abat_classical.argtypes = [_u64, _u64p, _sz, _sz, _sz, ctypes.POINTER(ctypes.c_int), _u64p, _u64p,
                                         _u64p, _sz, _u64p, _sz]
        L.orc_fp2_syrk_classical.argtypes = [_u64, _u64, _u64p, _sz, _sz, ctypes.c_int, _u64p]
        L.orc_syrkd.argtypes = [_u64, _u64p, _sz, _sz, _sz, _u64p, _u64p, _sz, _sz, _sz]
        L.orc_syrkd.restype = ctypes.c_long
        L.orc_level_blocks.argtypes = [_u64, _u64p, _sz, _sz, _sz, _sz, _sz] + [_u64p] * 9
        L.orc_dot_mod.argtypes = [_u64, _u64p, _u64p, _sz]
        L.orc_dot_mod.restype = _u64
        L.orc_lower_digest.argtypes = [_u64p, _sz, _sz, ctypes.c_char_p]
        _lib = L
    return _lib


UNLIMITED = (1 << 64) - 1


def _p(a):
    return a.ctypes.data_as(_u64p)


def mt64_stream(seed, count):
    out = np.empty(count, dtype=np.uint64)
    lib().orc_mt64_stream(seed, count, _p(out))
    return out


def random_matrix(p, rows, cols, seed):
    out = np.empty((rows, cols), dtype=np.uint64)
    lib().orc_random_matrix(p, rows, cols, seed, _p(out))
    return out


def random_nonzero(p, count, seed):
    out = np.empty(count, dtype=np.uint64)
    lib().orc_random_nonzero(p, count, seed, _p(out))
    return out


def alpha_beta(p, abseed):
    a, b = _u64(0), _u64(0)
    lib().orc_alpha_beta(p, abseed, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def skew(p):
    form, yc = ctypes.c_int(0), ctypes.c_int(0)
    a, b = _u64(0), _u64(0)
    lib().orc_skew(p, ctypes.byref(form), ctypes.byref(a), ctypes.byref(b), ctypes.byref(yc))
    return form.value, a.value, b.value, yc.value


def syrk_classical(p, a, alpha=1, beta=0, c=None):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    n, k = a.shape
    c = np.zeros((n, n), dtype=np.uint64) if c is None else c.copy()
    lib().orc_syrk_classical(p, alpha, _p(a), n, k, max(k, 1), beta, _p(c), max(n, 1))
    return c


def syrk_fast(p, a, threshold=64, levels=UNLIMITED):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    n, k = a.shape
    c = np.zeros((n, n), dtype=np.uint64)
    lib().orc_syrk_fast(p, _p(a), n, k, max(k, 1), _p(c), max(n, 1), threshold, levels)
    return c


def syrk_fast_acc(p, alpha, a, beta, c0, threshold=64, levels=UNLIMITED):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    n, k = a.shape
    c = np.ascontiguousarray(c0, dtype=np.uint64).copy()
    lib().orc_syrk_fast_acc(p, alpha, _p(a), n, k, max(k, 1), beta, _p(c), max(n, 1), threshold, levels)
    return c


def syrkd(p, a, d, threshold=64, levels=UNLIMITED):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    d = np.ascontiguousarray(d, dtype=np.uint64)
    n, k = a.shape
    c = np.zeros((n, n), dtype=np.uint64)
    kb = lib().orc_syrkd(p, _p(a), n, k, max(k, 1), _p(d), _p(c), max(n, 1), threshold, levels)
    if kb < 0:
        raise ValueError("syrkd failed")
    return c


def level_blocks(p, a):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    n, k = a.shape
    h = n // 2
    kw = k // 2 + 1
    S = [np.zeros((h, kw), dtype=np.uint64) for _ in range(4)]
    P = [np.zeros((h, h), dtype=np.uint64) for _ in range(5)]
    padded = lib().orc_level_blocks(p, _p(a), n, k, k, 2, 1, *[_p(s) for s in S], *[_p(x) for x in P])
    kw = k // 2 + (1 if padded == 1 else 0)
    S = [np.ascontiguousarray(s.reshape(-1)[: h * kw].reshape(h, kw)) for s in S]
    return {"S1": S[0], "S2": S[1], "S3": S[2], "S4": S[3],
            "P1": P[0], "P2": P[1], "P3": P[2], "P4": P[3], "P5": P[4], "kw": kw}


def dot_mod(p, x, y):
    x = np.ascontiguousarray(x, dtype=np.uint64)
    y = np.ascontiguousarray(y, dtype=np.uint64)
    return int(lib().orc_dot_mod(p, _p(x), _p(y), x.shape[0]))


def lower_digest(c):
    """SHA-256 of Low(C) as little-endian uint64, row by row (oracle/sha256.h)."""
    h = hashlib.sha256()
    n = c.shape[0]
    for i in range(n):
        h.update(np.ascontiguousarray(c[i, : i + 1], dtype="<u8").tobytes())
    return h.hexdigest()


def lower_equal(x, y):
    n = x.shape[0]
    idx = np.tril_indices(n)
    return x.shape == y.shape and np.array_equal(x[idx], y[idx])


def abat_classical(p, a, blocks):
    """Full (A B A^T) mod p for block-diagonal B given as [(two, d, beta, gamma), ...]
    (abat_oracle, test_scaled_syrk.cpp:25-47)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    n, k = a.shape
    nb = len(blocks)
    two = (ctypes.c_int * max(nb, 1))(*[int(b[0]) for b in blocks])
    cols = [np.ascontiguousarray(np.array([int(b[i]) for b in blocks] or [0], dtype=np.uint64)) for i in (1, 2, 3)]
    c = np.zeros((n, n), dtype=np.uint64)
    if n and k:
        lib().orc_abat_classical(p, _p(a), n, k, k, two, _p(cols[0]), _p(cols[1]), _p(cols[2]), nb, _p(c), n)
    return c


def lqnr(p):
    """Least quadratic non-residue (the QuadExtField modulus x^2 - ns, fields.hpp:148-150)."""
    return int(lib().orc_lqnr(p))


def fp2_syrk_classical(p, a_pairs, conj):
    """Lower triangle of A * conj(A)^T (conj) or A * A^T over F_{p^2}; a_pairs: (n, k, 2) uint64."""
    a = np.ascontiguousarray(a_pairs, dtype=np.uint64)
    n, k = a.shape[0], a.shape[1]
    c = np.zeros((n, n, 2), dtype=np.uint64)
    if n and k:
        lib().orc_fp2_syrk_classical(p, lqnr(p), _p(a), n, k, 1 if conj else 0, _p(c))
    return c
