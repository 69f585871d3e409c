"""Python mirror of the reference fsyrk PrimeField SYRK interface over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(paths relative to /root/reference/proj):

    PrimeField(p)                        include/fsyrk/fields.hpp:32-93
    RecursionPolicy(threshold, levels)   include/fsyrk/winograd.hpp:14-21
    OpCount                              include/fsyrk/opcount.hpp:10-25
    SkewOrthogonal / skew_orthogonal     include/fsyrk/skew.hpp:21-37, 66-73
    SyrkPlan / make_syrk_plan            include/fsyrk/fast_syrk.hpp:12-24
    syrk_fast_into / syrk_fast           include/fsyrk/fast_syrk.hpp:274-289
    syrk_fast_acc                        include/fsyrk/fast_syrk.hpp:293-303
    syrkd                                include/fsyrk/scaled_syrk.hpp:58-104
    random_matrix                        include/fsyrk/matrix.hpp:411-419

Matrices are numpy uint64 arrays with row-major rows (a row stride in
elements is allowed, as for the reference's views).  Every compute call runs
on the B200 through libfsyrk_b200.so; there is no CPU fallback -- without
the library or a device the calls raise.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSYRK_B200_LIB selects a tuning variant built by build.py --out (experiments only)
_LIB_PATH = os.environ.get("FSYRK_B200_LIB") or os.path.join(_HERE, "libfsyrk_b200.so")

UNLIMITED_LEVELS = (1 << 64) - 1  # kUnlimitedLevels, winograd.hpp:9


# ----------------------------------------------------------------- errors
class DimensionError(ValueError):
    """fsyrk::DimensionError (fields.hpp:21-23)."""


class DimensionParityError(ValueError):
    """fsyrk::DimensionParityError (fields.hpp:25-27)."""


class NotNonResidueError(ArithmeticError):
    """fsyrk::NotNonResidueError (fields.hpp:17-19)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL / missing-device failures (no reference analogue)."""


_STATUS = {
    1: DimensionError,
    2: ValueError,  # std::invalid_argument
    3: DimensionParityError,
    4: NotNonResidueError,
    5: ArithmeticError,  # std::domain_error
    6: DeviceError,
    7: MemoryError,
    8: DeviceError,
    9: DeviceError,
}


# ------------------------------------------------------------------ C ABI
class _Policy(ctypes.Structure):
    _fields_ = [("threshold", ctypes.c_uint64), ("max_levels", ctypes.c_uint64)]


class _OpCount(ctypes.Structure):
    _fields_ = [("mults", ctypes.c_uint64), ("adds", ctypes.c_uint64)]


class _Skew(ctypes.Structure):
    _fields_ = [("form", ctypes.c_int), ("a", ctypes.c_uint64), ("b", ctypes.c_uint64), ("ycost", ctypes.c_int)]


class _Block(ctypes.Structure):
    _fields_ = [("two", ctypes.c_int), ("d", ctypes.c_uint64), ("beta", ctypes.c_uint64), ("gamma", ctypes.c_uint64)]


_u64p = ctypes.POINTER(ctypes.c_uint64)
_lib = None

EXPORTS = (
    "fsyrk_b200_last_error", "fsyrk_b200_abi_version", "fsyrk_b200_device_available",
    "fsyrk_b200_make_syrk_plan", "fsyrk_b200_skew_orthogonal", "fsyrk_b200_random_matrix",
    "fsyrk_b200_syrk_fast_into", "fsyrk_b200_syrk_fast_acc", "fsyrk_b200_syrkd", "fsyrk_b200_syrk_dev",
    "fsyrk_b200_release_cache", "fsyrk_b200_last_launch_count", "fsyrk_b200_last_plan_json",
    "fsyrk_b200_set_phase_timing", "fsyrk_b200_last_phase_ms", "fsyrk_b200_level_blocks", "fsyrk_b200_gemm_nt",
    "fsyrk_b200_syrk_part_dev", "fsyrk_b200_partition_owners", "fsyrk_b200_syrkbd", "fsyrk_b200_syrkbd_dev",
    "fsyrk_b200_last_transfer_bytes", "fsyrk_b200_sum_of_squares", "fsyrk_b200_nrsyf",
    "fsyrk_b200_herk_fast_into", "fsyrk_b200_syrk_fast_into_fp2", "fsyrk_b200_gemm_winograd_nt",
    "fsyrk_b200_gemm_winograd_nt_dev", "fsyrk_b200_hostio_roundtrip", "fsyrk_b200_upload", "fsyrk_b200_download",
    "fsyrk_b200_syrk_mgpu", "fsyrk_b200_nccl_unique_id", "fsyrk_b200_comm_init_rank", "fsyrk_b200_comm_destroy",
    "fsyrk_b200_syrk_mgpu_rank", "fsyrk_b200_share_pairs", "fsyrk_b200_opcount_syrk", "fsyrk_b200_opcount_syrkd",
    "fsyrk_b200_opcount_syrkbd", "fsyrk_b200_opcount_fp2", "fsyrk_b200_workspace_bytes",
    "fsyrk_b200_set_workspace_limit", "fsyrk_b200_set_low_memory", "fsyrk_b200_set_winograd_min",
)


def lib() -> ctypes.CDLL:
    """Load libfsyrk_b200.so (built by paper_2001_04109_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_2001_04109_b200.build` "
                          "(the product path has no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    L.fsyrk_b200_last_error.restype = ctypes.c_char_p
    L.fsyrk_b200_last_plan_json.restype = ctypes.c_char_p
    L.fsyrk_b200_make_syrk_plan.argtypes = [ctypes.c_uint64, _Policy, ctypes.c_int, ctypes.POINTER(_Skew)]
    L.fsyrk_b200_skew_orthogonal.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.POINTER(_Skew)]
    L.fsyrk_b200_random_matrix.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64,
                                           _u64p, ctypes.c_size_t]
    L.fsyrk_b200_workspace_bytes.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, _Policy, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    L.fsyrk_b200_set_workspace_limit.argtypes = [ctypes.c_uint64]
    L.fsyrk_b200_set_low_memory.argtypes = [ctypes.c_int]
    L.fsyrk_b200_set_winograd_min.argtypes = [ctypes.c_uint64]
    L.fsyrk_b200_opcount_syrk.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64,
                                          ctypes.c_uint64, _Policy, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_opcount_syrkd.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, _u64p, ctypes.c_uint64,
                                           ctypes.c_uint64, _Policy, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_opcount_syrkbd.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.POINTER(_Block), ctypes.c_size_t,
                                            ctypes.c_uint64, ctypes.c_uint64, _Policy, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_opcount_fp2.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_size_t, _Policy,
                                         ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_syrk_fast_into.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t,
                                            ctypes.c_size_t, _u64p, ctypes.c_size_t, _Policy, ctypes.c_int,
                                            ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_syrk_fast_acc.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t,
                                           ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint64, _u64p,
                                           ctypes.c_size_t, _Policy, ctypes.c_int, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_syrkd.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t,
                                   ctypes.c_size_t, _u64p, ctypes.c_uint64, _u64p, ctypes.c_size_t, _Policy,
                                   ctypes.c_int, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_syrkbd.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t,
                                    ctypes.c_size_t, ctypes.POINTER(_Block), ctypes.c_size_t, ctypes.c_uint64, _u64p,
                                    ctypes.c_size_t, _Policy, ctypes.c_int, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_syrkbd_dev.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_size_t, ctypes.c_size_t, ctypes.POINTER(_Block), ctypes.c_size_t,
                                        ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t, _Policy, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_syrk_dev.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t,
                                      ctypes.c_size_t, ctypes.c_size_t, _u64p, ctypes.c_uint64, ctypes.c_void_p,
                                      ctypes.c_size_t, _Policy, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_syrk_part_dev.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t,
                                           ctypes.c_size_t, ctypes.c_size_t, _u64p, ctypes.c_uint64, ctypes.c_void_p,
                                           ctypes.c_size_t, _Policy, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_partition_owners.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_int,
                                              ctypes.POINTER(ctypes.c_int), ctypes.c_size_t,
                                              ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]
    L.fsyrk_b200_last_transfer_bytes.argtypes = [_u64p, _u64p]
    L.fsyrk_b200_syrk_mgpu.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t,
                                       ctypes.c_size_t, _u64p, ctypes.c_uint64, _u64p, ctypes.c_size_t, _Policy,
                                       ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                       ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.fsyrk_b200_comm_init_rank.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_void_p)]
    L.fsyrk_b200_comm_destroy.argtypes = [ctypes.c_void_p]
    L.fsyrk_b200_syrk_mgpu_rank.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_size_t,
                                            ctypes.c_size_t, ctypes.c_size_t, _u64p, ctypes.c_uint64, _u64p,
                                            ctypes.c_size_t, _Policy, ctypes.c_int, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_share_pairs.argtypes = [ctypes.c_uint64, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int), ctypes.c_size_t,
                                         ctypes.POINTER(ctypes.c_size_t)]
    L.fsyrk_b200_upload.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    L.fsyrk_b200_download.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                       ctypes.c_size_t, ctypes.c_int, _u64p, ctypes.c_size_t, ctypes.c_void_p]
    L.fsyrk_b200_hostio_roundtrip.argtypes = [_u64p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int,
                                              ctypes.c_int, _u64p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t),
                                              ctypes.POINTER(ctypes.c_double)]
    L.fsyrk_b200_gemm_winograd_nt.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t,
                                              ctypes.c_size_t, _u64p, ctypes.c_size_t, ctypes.c_size_t, _u64p,
                                              ctypes.c_size_t, _Policy]
    L.fsyrk_b200_gemm_winograd_nt_dev.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                                  ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                                  ctypes.c_void_p, ctypes.c_size_t, _Policy, ctypes.c_void_p]
    for name in ("fsyrk_b200_herk_fast_into", "fsyrk_b200_syrk_fast_into_fp2"):
        getattr(L, name).argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                     _u64p, ctypes.c_size_t, _Policy, ctypes.c_int, ctypes.POINTER(_OpCount)]
    L.fsyrk_b200_sum_of_squares.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _u64p, _u64p]
    L.fsyrk_b200_nrsyf.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u64p]
    L.fsyrk_b200_last_launch_count.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    L.fsyrk_b200_last_phase_ms.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    L.fsyrk_b200_level_blocks.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t,
                                          ctypes.c_size_t] + [_u64p] * 9 + [ctypes.POINTER(ctypes.c_size_t)]
    L.fsyrk_b200_gemm_nt.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                     _u64p, ctypes.c_size_t, ctypes.c_size_t, _u64p, ctypes.c_size_t]
    _lib = L
    return L


def _check(status: int) -> None:
    if status != 0:
        msg = lib().fsyrk_b200_last_error().decode()
        raise _STATUS.get(status, RuntimeError)(msg)


def device_available() -> bool:
    return bool(lib().fsyrk_b200_device_available())


# -------------------------------------------------------------- the field
class PrimeField:
    """Z/pZ, 2 <= p < 2^31 prime (fields.hpp:32-93; validation fields.cpp:33-37)."""

    def __init__(self, p: int):
        p = int(p)
        if p >= 1 << 31:
            raise ValueError(f"prime modulus must be < 2^31, got {p}")
        if not _is_prime(p):
            raise ValueError(f"{p} is not prime")
        self.p = p

    def modulus(self) -> int:
        return self.p

    characteristic = modulus

    def zero(self) -> int:
        return 0

    def one(self) -> int:
        return 1

    def add(self, a: int, b: int) -> int:
        return (a + b) % self.p

    def sub(self, a: int, b: int) -> int:
        return (a - b) % self.p

    def neg(self, a: int) -> int:
        return (-a) % self.p

    def mul(self, a: int, b: int) -> int:
        return (a * b) % self.p

    def from_int(self, v: int) -> int:
        return int(v) % self.p

    def name(self) -> str:
        return f"F_{self.p}"


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    d = 3
    while d * d <= n:
        if n % d == 0:
            return False
        d += 2
    return True


@dataclass
class RecursionPolicy:
    threshold: int = 64
    max_levels: int = UNLIMITED_LEVELS

    def validate(self) -> None:
        if self.threshold < 2:
            raise ValueError("recursion threshold must be >= 2")

    def _c(self) -> _Policy:
        return _Policy(int(self.threshold), int(self.max_levels))


@dataclass
class OpCount:
    mults: int = 0
    adds: int = 0

    def total(self) -> int:
        return self.mults + self.adds


@dataclass
class SkewOrthogonal:
    form: str  # "scalar" | "pair"
    a: int
    b: int
    dim: int
    ycost: int


@dataclass
class SyrkPlan:
    policy: RecursionPolicy = field(default_factory=RecursionPolicy)
    skew: Optional[SkewOrthogonal] = None
    mirror_output: bool = False
    conjugate: bool = False  # herk plans (make_herk_plan, fast_syrk.hpp:17, 26-29)


def sum_of_squares(f: PrimeField, k: int):
    """(a, b) with a^2 + b^2 = k mod p (fields.cpp:114-123)."""
    a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(lib().fsyrk_b200_sum_of_squares(f.p, int(k) % f.p, ctypes.byref(a), ctypes.byref(b)))
    return int(a.value), int(b.value)


def nrsyf(f: PrimeField, alpha: int, beta: int):
    """[a, b, c, d] with [[a, b], [c, d]] [[a, b], [c, d]]^T = diag(alpha, beta) (skew.hpp:180-194)."""
    y = (ctypes.c_uint64 * 4)()
    _check(lib().fsyrk_b200_nrsyf(f.p, int(alpha) % f.p, int(beta) % f.p, y))
    return [int(v) for v in y]


def skew_orthogonal(f: PrimeField, dim: int) -> SkewOrthogonal:
    s = _Skew()
    _check(lib().fsyrk_b200_skew_orthogonal(f.p, int(dim), ctypes.byref(s)))
    return SkewOrthogonal("pair" if s.form == 1 else "scalar", s.a, s.b, int(dim), s.ycost)


def make_syrk_plan(f: PrimeField, policy: Optional[RecursionPolicy] = None, mirror_output: bool = False) -> SyrkPlan:
    policy = policy or RecursionPolicy()
    policy.validate()
    s = _Skew()
    _check(lib().fsyrk_b200_make_syrk_plan(f.p, policy._c(), int(bool(mirror_output)), ctypes.byref(s)))
    return SyrkPlan(policy, SkewOrthogonal("pair" if s.form == 1 else "scalar", s.a, s.b, 0, s.ycost),
                    bool(mirror_output))


# ------------------------------------------------------------ matrix glue
def _view(m: np.ndarray, name: str):
    if not isinstance(m, np.ndarray) or m.dtype != np.uint64 or m.ndim != 2:
        raise DimensionError(f"{name} must be a 2-D numpy uint64 array")
    if m.size > 0 and m.shape[1] > 1 and m.strides[1] != 8:
        raise DimensionError(f"{name} rows must be contiguous")
    if m.size > 0 and m.shape[0] > 1 and (m.strides[0] % 8 != 0 or m.strides[0] < 8 * m.shape[1]):
        # negative, overlapping or misaligned row strides cannot be expressed as a (data, ld)
        # view: the library would walk forward from the first row's address
        raise DimensionError(f"{name} row stride must be a positive multiple of 8 bytes >= 8*cols")
    ld = m.strides[0] // 8 if m.shape[0] > 1 and m.size > 0 else max(m.shape[1], 1)
    return m.ctypes.data_as(_u64p), int(m.shape[0]), int(m.shape[1]), int(ld)


def random_matrix(f: PrimeField, rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty((int(rows), int(cols)), dtype=np.uint64)
    _check(lib().fsyrk_b200_random_matrix(f.p, int(rows), int(cols), int(seed) & ((1 << 64) - 1),
                                          out.ctypes.data_as(_u64p), max(int(cols), 1)))
    return out


def _ops_out(ops: Optional[OpCount], c_ops: _OpCount) -> None:
    if ops is not None:
        ops.mults += c_ops.mults
        ops.adds += c_ops.adds


def syrk_fast_into(f: PrimeField, a: np.ndarray, c: np.ndarray, plan: SyrkPlan, ops: Optional[OpCount] = None) -> None:
    """Low(C) <- Low(A A^T) (fast_syrk.hpp:274-282)."""
    plan.policy.validate()
    pa, n, k, lda = _view(a, "a")
    pc, cn, cm, ldc = _view(c, "c")
    if cn != cm or cn != n:
        raise DimensionError("syrk_fast: dimension mismatch")
    co = _OpCount()
    _check(lib().fsyrk_b200_syrk_fast_into(f.p, pa, n, k, lda, pc, ldc, plan.policy._c(),
                                           int(plan.mirror_output), ctypes.byref(co)))
    _ops_out(ops, co)


def syrk_fast(f: PrimeField, a: np.ndarray, plan: SyrkPlan, ops: Optional[OpCount] = None) -> np.ndarray:
    """Returns a new C with Low(C) = Low(A A^T), zeros elsewhere (fast_syrk.hpp:284-289)."""
    c = np.zeros((a.shape[0], a.shape[0]), dtype=np.uint64)
    syrk_fast_into(f, a, c, plan, ops)
    return c


def syrk_fast_acc(f: PrimeField, alpha: int, a: np.ndarray, beta: int, c: np.ndarray, plan: SyrkPlan,
                  ops: Optional[OpCount] = None) -> None:
    """Low(C) <- Low(alpha A A^T + beta C) (fast_syrk.hpp:293-303)."""
    plan.policy.validate()
    pa, n, k, lda = _view(a, "a")
    pc, cn, cm, ldc = _view(c, "c")
    if cn != cm or cn != n:
        raise DimensionError("syrk_fast_acc: dimension mismatch")
    co = _OpCount()
    _check(lib().fsyrk_b200_syrk_fast_acc(f.p, int(alpha) % f.p, pa, n, k, lda, int(beta) % f.p, pc, ldc,
                                          plan.policy._c(), int(plan.mirror_output), ctypes.byref(co)))
    _ops_out(ops, co)


def syrkd(f: PrimeField, a: np.ndarray, d: Sequence[int], plan: SyrkPlan, ops: Optional[OpCount] = None,
          alpha: int = 1, beta: int = 0, c: Optional[np.ndarray] = None) -> np.ndarray:
    """Low(A Diag(d) A^T) (scaled_syrk.hpp:58-104); with alpha/beta/c it is the
    Schur-complement form Low(C) <- Low(alpha A D A^T + beta C) in one call."""
    plan.policy.validate()
    if f.p == 2:
        raise ValueError("syrkd requires an odd prime field")
    pa, n, k, lda = _view(a, "a")
    dv = np.ascontiguousarray(np.asarray(d, dtype=np.uint64))
    if dv.ndim != 1 or dv.shape[0] != k:
        raise DimensionError("syrkd: diagonal length must match column count")
    if c is None:
        c = np.zeros((n, n), dtype=np.uint64)
    pc, cn, cm, ldc = _view(c, "c")
    if cn != cm or cn != n:
        raise DimensionError("syrkd: dimension mismatch")
    co = _OpCount()
    dptr = dv.ctypes.data_as(_u64p) if k > 0 else None
    _check(lib().fsyrk_b200_syrkd(f.p, int(alpha) % f.p, pa, n, k, lda, dptr, int(beta) % f.p, pc, ldc,
                                  plan.policy._c(), int(plan.mirror_output), ctypes.byref(co)))
    _ops_out(ops, co)
    return c


@dataclass
class Block:
    """One block of BlockDiagonal (scaled_syrk.hpp:13-20): scalar d, or ((0, beta), (beta, gamma))."""
    two: bool = False
    d: int = 0
    beta: int = 0
    gamma: int = 0


@dataclass
class BlockDiagonal:
    """Middle matrix of A B A^T (scaled_syrk.hpp:12-37)."""
    blocks: list = field(default_factory=list)

    @staticmethod
    def scalar(d: int) -> Block:
        return Block(False, int(d), 0, 0)

    @staticmethod
    def two_by_two(beta: int, gamma: int) -> Block:
        return Block(True, 0, int(beta), int(gamma))

    def dimension(self) -> int:
        return sum(2 if b.two else 1 for b in self.blocks)

    def validate(self, f: PrimeField) -> None:
        for b in self.blocks:
            if b.two and b.beta % f.p == 0:
                raise ValueError("block-diagonal: 2x2 block requires beta != 0")

    def _c(self):
        arr = (_Block * max(len(self.blocks), 1))()
        for i, b in enumerate(self.blocks):
            arr[i] = _Block(int(b.two), int(b.d), int(b.beta), int(b.gamma))
        return arr


def syrkbd(f: PrimeField, a: np.ndarray, b: BlockDiagonal, plan: SyrkPlan, ops: Optional[OpCount] = None,
           alpha: int = 1, beta: int = 0, c: Optional[np.ndarray] = None) -> np.ndarray:
    """Low(A B A^T) for block-diagonal B (scaled_syrk.hpp:117-159); alpha/beta/c as in syrkd."""
    plan.policy.validate()
    b.validate(f)
    pa, n, k, lda = _view(a, "a")
    if b.dimension() != k:
        raise DimensionError("syrkbd: block-diagonal dimension must match column count")
    if f.p == 2:
        raise ValueError("syrkbd over characteristic 2 uses BinaryField")
    if c is None:
        c = np.zeros((n, n), dtype=np.uint64)
    pc, cn, cm, ldc = _view(c, "c")
    if cn != cm or cn != n:
        raise DimensionError("syrkbd: dimension mismatch")
    co = _OpCount()
    _check(lib().fsyrk_b200_syrkbd(f.p, int(alpha) % f.p, pa, n, k, lda, b._c(), len(b.blocks), int(beta) % f.p, pc,
                                   ldc, plan.policy._c(), int(plan.mirror_output), ctypes.byref(co)))
    _ops_out(ops, co)
    return c


def syrkbd_dev(p: int, alpha: int, a_ptr: int, n: int, k: int, lda: int, b: BlockDiagonal, beta: int, c_ptr: int,
               ldc: int, policy: RecursionPolicy, mirror: bool = False, stream: int = 0,
               ops: Optional[OpCount] = None) -> None:
    """Device-resident syrkbd (fsyrk_b200_syrkbd_dev)."""
    co = _OpCount()
    _check(lib().fsyrk_b200_syrkbd_dev(int(p), int(alpha) % p, ctypes.c_void_p(a_ptr), int(n), int(k), int(lda),
                                       b._c(), len(b.blocks), int(beta) % p, ctypes.c_void_p(c_ptr), int(ldc),
                                       policy._c(), int(mirror), ctypes.c_void_p(stream), ctypes.byref(co)))
    _ops_out(ops, co)


class QuadExtField:
    """F_{p^2} = F_p[x] / (x^2 - ns), ns the least quadratic non-residue (fields.hpp:148-212).
    Matrices over it are numpy uint64 arrays of shape (rows, cols, 2): (a, b) = a + b x."""

    def __init__(self, p: int):
        self.base = PrimeField(p)
        if self.base.p == 2:
            raise ValueError("QuadExtField requires an odd prime")
        self.p = self.base.p

    def characteristic(self) -> int:
        return self.p

    def name(self) -> str:
        return f"F_{self.p}^2"


def _view_fp2(m: np.ndarray, name: str):
    if not isinstance(m, np.ndarray) or m.dtype != np.uint64 or m.ndim != 3 or m.shape[2] != 2:
        raise DimensionError(f"{name} must be a (rows, cols, 2) numpy uint64 array of (a, b) pairs")
    if m.size > 0 and (m.strides[2] != 8 or (m.shape[1] > 1 and m.strides[1] != 16)):
        raise DimensionError(f"{name} rows must be contiguous pairs")
    if m.size > 0 and m.shape[0] > 1 and (m.strides[0] % 16 != 0 or m.strides[0] < 16 * m.shape[1]):
        raise DimensionError(f"{name} row stride must be a positive multiple of 16 bytes >= 16*cols")
    ld = m.strides[0] // 16 if m.shape[0] > 1 and m.size > 0 else max(m.shape[1], 1)
    return m.ctypes.data_as(_u64p), int(m.shape[0]), int(m.shape[1]), int(ld)


def make_herk_plan(f: QuadExtField, policy: Optional[RecursionPolicy] = None, mirror_output: bool = False) -> SyrkPlan:
    """make_herk_plan (fast_syrk.hpp:26-29): a conjugating plan."""
    policy = policy or RecursionPolicy()
    policy.validate()
    return SyrkPlan(policy, None, bool(mirror_output), True)


def _fp2_call(fn, f: QuadExtField, a: np.ndarray, c: np.ndarray, plan: SyrkPlan, ops: Optional[OpCount]):
    plan.policy.validate()
    pa, n, k, lda = _view_fp2(a, "a")
    pc, cn, cm, ldc = _view_fp2(c, "c")
    if cn != cm or cn != n:
        raise DimensionError("syrk_fast: dimension mismatch")
    co = _OpCount()
    _check(fn(f.p, pa, n, k, lda, pc, ldc, plan.policy._c(), int(plan.mirror_output), ctypes.byref(co)))
    _ops_out(ops, co)


def herk_fast_into(f: QuadExtField, a: np.ndarray, c: np.ndarray, plan: SyrkPlan, ops: Optional[OpCount] = None):
    """Low(C) <- Low(A conj(A)^T) over F_{p^2} (fast_syrk.hpp:307-313)."""
    if not getattr(plan, "conjugate", False):
        raise ValueError("herk_fast: plan must be built by make_herk_plan")
    _fp2_call(lib().fsyrk_b200_herk_fast_into, f, a, c, plan, ops)


def herk_fast(f: QuadExtField, a: np.ndarray, plan: SyrkPlan, ops: Optional[OpCount] = None) -> np.ndarray:
    c = np.zeros((a.shape[0], a.shape[0], 2), dtype=np.uint64)
    herk_fast_into(f, a, c, plan, ops)
    return c


def syrk_fast_fp2(f: QuadExtField, a: np.ndarray, plan: SyrkPlan, ops: Optional[OpCount] = None) -> np.ndarray:
    """Low(A A^T) over F_{p^2} (syrk_fast, fast_syrk.hpp:284-289, for QuadExtField)."""
    c = np.zeros((a.shape[0], a.shape[0], 2), dtype=np.uint64)
    _fp2_call(lib().fsyrk_b200_syrk_fast_into_fp2, f, a, c, plan, ops)
    return c


def syrk_dev(p: int, alpha: int, a_ptr: int, n: int, k: int, lda: int, beta: int, c_ptr: int, ldc: int,
             policy: RecursionPolicy, mirror: bool = False, stream: int = 0, d: Optional[np.ndarray] = None,
             ops: Optional[OpCount] = None) -> None:
    """Device-resident form (fsyrk_b200_syrk_dev): a_ptr / c_ptr are CUDA device
    pointers to uint64 matrices; stream is a cudaStream_t handle."""
    co = _OpCount()
    dptr = None
    if d is not None:
        dv = np.ascontiguousarray(np.asarray(d, dtype=np.uint64))
        dptr = dv.ctypes.data_as(_u64p)
    _check(lib().fsyrk_b200_syrk_dev(int(p), int(alpha) % p, ctypes.c_void_p(a_ptr), int(n), int(k), int(lda), dptr,
                                     int(beta) % p, ctypes.c_void_p(c_ptr), int(ldc), policy._c(), int(mirror),
                                     ctypes.c_void_p(stream), ctypes.byref(co)))
    _ops_out(ops, co)


def syrk_part_dev(p: int, alpha: int, a_ptr: int, n: int, k: int, lda: int, beta: int, c_ptr: int, ldc: int,
                  policy: RecursionPolicy, rank: int, nranks: int, stream: int = 0, d: Optional[np.ndarray] = None,
                  ops: Optional[OpCount] = None) -> None:
    """One rank's share of a multi-GPU call (fsyrk_b200_syrk_part_dev): the entries of Low(C)
    in the top-level block pairs owned by `rank`; the union over ranks is the full result."""
    co = _OpCount()
    dptr = None
    if d is not None:
        dv = np.ascontiguousarray(np.asarray(d, dtype=np.uint64))
        dptr = dv.ctypes.data_as(_u64p)
    _check(lib().fsyrk_b200_syrk_part_dev(int(p), int(alpha) % p, ctypes.c_void_p(a_ptr), int(n), int(k), int(lda),
                                          dptr, int(beta) % p, ctypes.c_void_p(c_ptr), int(ldc), policy._c(),
                                          int(rank), int(nranks), ctypes.c_void_p(stream), ctypes.byref(co)))
    _ops_out(ops, co)


def partition_owners(p: int, h: int, nranks: int):
    """Owner rank of each top-level block pair (I >= J) as an nb x nb array (-1 above the
    diagonal), and the block size in rows."""
    nb, blk = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _check(lib().fsyrk_b200_partition_owners(int(p), int(h), int(nranks), None, 0, ctypes.byref(nb),
                                             ctypes.byref(blk)))
    out = np.full(nb.value * nb.value, -1, dtype=np.int32)
    _check(lib().fsyrk_b200_partition_owners(int(p), int(h), int(nranks),
                                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), out.size,
                                             ctypes.byref(nb), ctypes.byref(blk)))
    return out.reshape(nb.value, nb.value), blk.value


def gemm_nt(f: PrimeField, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """C = A B^T mod p on the tensor cores (gemm_classical_nt, matrix.hpp:317-329)."""
    pa, m, k, lda = _view(a, "a")
    pb, n, kb, ldb = _view(b, "b")
    if kb != k:
        raise DimensionError("gemm_nt: dimension mismatch")
    c = np.zeros((m, n), dtype=np.uint64)
    _check(lib().fsyrk_b200_gemm_nt(f.p, pa, m, k, lda, pb, n, ldb, c.ctypes.data_as(_u64p), max(n, 1)))
    return c


def gemm_winograd_nt(f: PrimeField, a: np.ndarray, b: np.ndarray, policy: Optional[RecursionPolicy] = None) -> np.ndarray:
    """C = A B^T by Strassen-Winograd levels over the tensor-core product (winograd.hpp:195-202)."""
    policy = policy or RecursionPolicy()
    policy.validate()
    pa, m, k, lda = _view(a, "a")
    pb, n, kb, ldb = _view(b, "b")
    if kb != k:
        raise DimensionError("gemm_winograd_nt: dimension mismatch")
    c = np.zeros((m, n), dtype=np.uint64)
    pc, _, _, ldc = _view(c, "c")
    _check(lib().fsyrk_b200_gemm_winograd_nt(f.p, pa, m, k, lda, pb, n, ldb, pc, ldc, policy._c()))
    return c


def gemm_winograd_nt_dev(p: int, a_ptr: int, m: int, k: int, lda: int, b_ptr: int, n: int, ldb: int, c_ptr: int,
                         ldc: int, policy: RecursionPolicy, stream: int = 0) -> None:
    _check(lib().fsyrk_b200_gemm_winograd_nt_dev(int(p), ctypes.c_void_p(a_ptr), int(m), int(k), int(lda),
                                                 ctypes.c_void_p(b_ptr), int(n), int(ldb), ctypes.c_void_p(c_ptr),
                                                 int(ldc), policy._c(), ctypes.c_void_p(stream)))


def level_blocks(f: PrimeField, a: np.ndarray):
    """White-box: the S1..S4 and P1..P5 blocks of one device recursion level."""
    pa, n, k, lda = _view(a, "a")
    h = n // 2
    kw = k // 2 + 1
    S = [np.zeros((h, kw), dtype=np.uint64) for _ in range(4)]
    P = [np.zeros((h, h), dtype=np.uint64) for _ in range(5)]
    kw_out = ctypes.c_size_t(0)
    _check(lib().fsyrk_b200_level_blocks(f.p, pa, n, k, lda, *[s.ctypes.data_as(_u64p) for s in S],
                                         *[x.ctypes.data_as(_u64p) for x in P], ctypes.byref(kw_out)))
    kw = kw_out.value
    S = [np.ascontiguousarray(s.reshape(-1)[: h * kw].reshape(h, kw)) for s in S]
    return {"S1": S[0], "S2": S[1], "S3": S[2], "S4": S[3],
            "P1": P[0], "P2": P[1], "P3": P[2], "P4": P[3], "P5": P[4], "kw": kw}


def workspace_bytes(p: int, n: int, k: int, policy: Optional[RecursionPolicy] = None, lowmem: bool = False) -> dict:
    """Device memory of a call without allocating it (host only): the plan's workspace (wide or
    low-memory schedule) and, for the host entry points, workspace + device staging of A and C."""
    ar, hc = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(lib().fsyrk_b200_workspace_bytes(int(p), int(n), int(k), (policy or RecursionPolicy())._c(), int(lowmem),
                                            ctypes.byref(ar), ctypes.byref(hc)))
    return {"arena": int(ar.value), "host_call": int(hc.value)}


def set_workspace_limit(nbytes: int) -> None:
    """Process-wide workspace limit (0 = none): larger plans run the low-memory schedule."""
    _check(lib().fsyrk_b200_set_workspace_limit(int(nbytes)))


def set_winograd_min(min_dim: int) -> None:
    """Process-wide: top-level general products with min(h, kw) >= min_dim run Strassen-Winograd
    levels (0 = never; default 16384)."""
    _check(lib().fsyrk_b200_set_winograd_min(int(min_dim)))


def set_low_memory(enable: bool) -> None:
    """Process-wide: run every plan created afterwards with the low-memory schedule."""
    _check(lib().fsyrk_b200_set_low_memory(int(bool(enable))))


def reference_opcount(p: int, n: int, k: int, policy: Optional[RecursionPolicy] = None, alpha: int = 1, beta: int = 0,
                      d: Optional[Sequence[int]] = None, blocks: Optional[BlockDiagonal] = None,
                      fp2: bool = False) -> OpCount:
    """The OpCount the reference adds for one call (host only, no device): syrk_fast_into /
    syrk_fast_acc (fast_syrk.hpp:274-303), syrkd with `d` (scaled_syrk.hpp:58-104), syrkbd with
    `blocks` (:117-159), or herk/syrk over F_{p^2} with fp2=True (fast_syrk.hpp:305-320).
    The library's entry points fill their `ops` argument with exactly this."""
    pol = (policy or RecursionPolicy())._c()
    c = _OpCount()
    if fp2:
        _check(lib().fsyrk_b200_opcount_fp2(int(p), int(n), int(k), pol, ctypes.byref(c)))
    elif blocks is not None:
        arr = blocks._c()
        _check(lib().fsyrk_b200_opcount_syrkbd(int(p), int(n), arr, len(blocks.blocks), int(alpha), int(beta), pol,
                                               ctypes.byref(c)))
    elif d is not None:
        dv = np.ascontiguousarray(np.asarray(d, dtype=np.uint64))
        _check(lib().fsyrk_b200_opcount_syrkd(int(p), int(n), len(dv), dv.ctypes.data_as(_u64p), int(alpha),
                                              int(beta), pol, ctypes.byref(c)))
    else:
        _check(lib().fsyrk_b200_opcount_syrk(int(p), int(n), int(k), int(alpha), int(beta), pol, ctypes.byref(c)))
    return OpCount(int(c.mults), int(c.adds))


def last_launch_counts() -> dict:
    arr = (ctypes.c_int * 5)()
    total = lib().fsyrk_b200_last_launch_count(arr, 5)
    return {"total": total, "products": arr[0], "pre": arr[1], "post": arr[2], "convert": arr[3], "other": arr[4]}


def last_transfer_bytes() -> tuple:
    """(host->device, device->host) bytes of the last host-API call on this thread."""
    h, d = ctypes.c_uint64(0), ctypes.c_uint64(0)
    lib().fsyrk_b200_last_transfer_bytes(ctypes.byref(h), ctypes.byref(d))
    return int(h.value), int(d.value)


def transfer_bits(p: int) -> int:
    """Width of a residue on the wire for the host entry points (host_io.cu transfer_bits)."""
    b = max(8, (int(p) - 1).bit_length())
    return b if b <= 24 and os.environ.get("FSYRK_B200_PACK", "1") != "0" else 32


def upload(p: int, h: np.ndarray, d_ptr: int, ldd: int, lower: bool = False, stream: int = 0) -> None:
    """Host rows -> device uint64 rows through the library's staging path (fsyrk_b200_upload)."""
    ph, rows, cols, ldh = _view(h, "h")
    _check(lib().fsyrk_b200_upload(int(p), ph, rows, cols, ldh, int(bool(lower)), ctypes.c_void_p(d_ptr), int(ldd),
                                   ctypes.c_void_p(stream)))


def download(p: int, d_ptr: int, ldd: int, h: np.ndarray, lower: bool = False, stream: int = 0) -> None:
    """Device uint64 rows (residues) -> host rows (fsyrk_b200_download; synchronous)."""
    ph, rows, cols, ldh = _view(h, "h")
    _check(lib().fsyrk_b200_download(int(p), ctypes.c_void_p(d_ptr), rows, cols, int(ldd), int(bool(lower)), ph, ldh,
                                     ctypes.c_void_p(stream)))


def hostio_roundtrip(a: np.ndarray, lower: bool, bits: int):
    """Host-only pack -> unpack of `a`'s rows (lower: row i holds columns [0, i]) in the host
    transfer format (fsyrk_b200_hostio_roundtrip).  Returns (out, raw_chunks, (pack_s, unpack_s));
    entries outside the region stay zero."""
    pa, rows, cols, lda = _view(a, "a")
    out = np.zeros((rows, cols), dtype=np.uint64)
    raw = ctypes.c_size_t(0)
    secs = (ctypes.c_double * 2)()
    _check(lib().fsyrk_b200_hostio_roundtrip(pa, rows, cols, lda, int(bool(lower)), int(bits),
                                             out.ctypes.data_as(_u64p), max(cols, 1), ctypes.byref(raw), secs))
    return out, int(raw.value), (secs[0], secs[1])


def last_plan() -> dict:
    s = lib().fsyrk_b200_last_plan_json().decode()
    return json.loads(s) if s else {}


def set_phase_timing(enable: bool) -> None:
    lib().fsyrk_b200_set_phase_timing(int(enable))


def last_phase_ms() -> dict:
    arr = (ctypes.c_float * 5)()
    lib().fsyrk_b200_last_phase_ms(arr, 5)
    return {"products": arr[0], "pre": arr[1], "post": arr[2], "convert": arr[3]}


def release_cache() -> None:
    lib().fsyrk_b200_release_cache()


# -------------------------------------------------------------- multi-GPU
def _mgpu_args(f: PrimeField, a: np.ndarray, c: np.ndarray, d):
    pa, n, k, lda = _view(a, "a")
    pc, cn, cm, ldc = _view(c, "c")
    if cn != cm or cn != n:
        raise DimensionError("syrk_fast: dimension mismatch")
    dptr, keep = None, None
    if d is not None:
        keep = np.ascontiguousarray(np.asarray(d, dtype=np.uint64))
        if keep.ndim != 1 or keep.shape[0] != k:
            raise DimensionError("syrkd: diagonal length must match column count")
        dptr = keep.ctypes.data_as(_u64p) if k > 0 else None
    return pa, n, k, lda, pc, ldc, dptr, keep


def syrk_mgpu(f: PrimeField, a: np.ndarray, c: np.ndarray, plan: SyrkPlan, devices: Sequence[int], alpha: int = 1,
              beta: int = 0, d: Optional[np.ndarray] = None, ops: Optional[OpCount] = None) -> np.ndarray:
    """Multi-GPU Low(C) <- Low(alpha A Diag(d) A^T + beta C) over `devices` of this process
    (fsyrk_b200_syrk_mgpu: NCCL broadcast of A, owned tile pairs per device, uint32 share gather)."""
    plan.policy.validate()
    pa, n, k, lda, pc, ldc, dptr, _keep = _mgpu_args(f, a, c, d)
    devs = (ctypes.c_int * max(1, len(devices)))(*[int(x) for x in devices])
    co = _OpCount()
    _check(lib().fsyrk_b200_syrk_mgpu(f.p, int(alpha) % f.p, pa, n, k, lda, dptr, int(beta) % f.p, pc, ldc,
                                      plan.policy._c(), int(plan.mirror_output), devs, len(devices), ctypes.byref(co)))
    _ops_out(ops, co)
    return c


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().fsyrk_b200_nccl_unique_id(buf))
    return buf.raw


class Communicator:
    """One rank of a multi-process (one process per GPU) library call: the NCCL communicator
    on the current device (fsyrk_b200_comm_init_rank)."""

    def __init__(self, uid: bytes, rank: int, nranks: int):
        h = ctypes.c_void_p()
        _check(lib().fsyrk_b200_comm_init_rank(bytes(uid), int(rank), int(nranks), ctypes.byref(h)))
        self.handle, self.rank, self.nranks = h, int(rank), int(nranks)

    def close(self) -> None:
        if self.handle:
            _check(lib().fsyrk_b200_comm_destroy(self.handle))
            self.handle = None

    def syrk(self, f: PrimeField, a: Optional[np.ndarray], c: Optional[np.ndarray], n: int, k: int, plan: SyrkPlan,
             alpha: int = 1, beta: int = 0, d: Optional[np.ndarray] = None, ops: Optional[OpCount] = None) -> None:
        """Collective fsyrk_b200_syrk_mgpu_rank: rank 0 passes host a (n x k) and c (n x n);
        the other ranks pass None."""
        plan.policy.validate()
        if self.rank == 0:
            pa, n2, k2, lda, pc, ldc, dptr, _keep = _mgpu_args(f, a, c, d)
            if (n2, k2) != (int(n), int(k)):
                raise DimensionError("syrk_mgpu: dimension mismatch")
        else:
            pa = pc = None
            lda, ldc = max(int(k), 1), max(int(n), 1)
            _keep = None if d is None else np.ascontiguousarray(np.asarray(d, dtype=np.uint64))
            dptr = _keep.ctypes.data_as(_u64p) if _keep is not None and int(k) > 0 else None
        co = _OpCount()
        _check(lib().fsyrk_b200_syrk_mgpu_rank(self.handle, f.p, int(alpha) % f.p, pa, int(n), int(k), lda, dptr,
                                               int(beta) % f.p, pc, ldc, plan.policy._c(), int(plan.mirror_output),
                                               ctypes.byref(co)))
        _ops_out(ops, co)


def share_pairs(p: int, h: int, rank: int, nranks: int) -> np.ndarray:
    """Tile pairs (I, J) of rank's share of Low(C) (fsyrk_b200_share_pairs), shape (count, 2)."""
    cnt = ctypes.c_size_t(0)
    _check(lib().fsyrk_b200_share_pairs(int(p), int(h), int(rank), int(nranks), None, 0, ctypes.byref(cnt)))
    out = np.zeros((cnt.value, 2), dtype=np.int32)
    _check(lib().fsyrk_b200_share_pairs(int(p), int(h), int(rank), int(nranks),
                                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), cnt.value,
                                        ctypes.byref(cnt)))
    return out
