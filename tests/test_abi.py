"""C-ABI boundary checks that need no GPU: the library builds, loads, exports
every symbol include/fsyrk_b200.h declares, validates like the reference,
and refuses to compute without a device (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle_py as orc

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(REPO, "include", "fsyrk_b200.h")).read()
    return sorted(set(re.findall(r"\b(fsyrk_b200_[a-z0-9_]+)\s*\(", hdr)))


def test_header_and_exports(fsyrk):
    lib = fsyrk.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(fsyrk.fsyrk.EXPORTS)
    assert lib.fsyrk_b200_abi_version() == 1


def test_random_matrix_matches_reference(fsyrk, golden):
    for case in golden["cases"][:20]:
        f = fsyrk.PrimeField(case["p"])
        a = fsyrk.random_matrix(f, case["n"], case["k"], case["seed"])
        assert np.array_equal(a, case["A"])


def test_skew_and_plan(fsyrk, golden):
    for p, form, a, b in zip(golden["skew_p"], golden["skew_form"], golden["skew_a"], golden["skew_b"]):
        f = fsyrk.PrimeField(int(p))
        y = fsyrk.skew_orthogonal(f, 2)
        assert (y.form == "pair", y.a, y.b) == (bool(form), int(a), int(b))
        plan = fsyrk.make_syrk_plan(f, fsyrk.RecursionPolicy(2))
        assert plan.skew.a == int(a)
    # 2x2 over F_5: plan.skew.a == 2 (test_fast_syrk.cpp:54-69)
    assert fsyrk.make_syrk_plan(fsyrk.PrimeField(5), fsyrk.RecursionPolicy(2)).skew.a == 2


def test_validation_errors(fsyrk):
    with pytest.raises(ValueError):
        fsyrk.PrimeField(4)
    with pytest.raises(ValueError):
        fsyrk.PrimeField(1 << 31)
    f = fsyrk.PrimeField(7)
    with pytest.raises(ValueError):
        fsyrk.make_syrk_plan(f, fsyrk.RecursionPolicy(1))
    with pytest.raises(fsyrk.DimensionParityError):
        fsyrk.skew_orthogonal(fsyrk.PrimeField(11), 5)
    # C-level validation happens before any device work
    lib = fsyrk.lib()
    a = np.ones((8, 8), dtype=np.uint64)
    pol = fsyrk.fsyrk._Policy(2, 1 << 63)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    st = lib.fsyrk_b200_syrk_fast_into(7, a.ctypes.data_as(u64p), 8, 8, 8, a.ctypes.data_as(u64p), 8, pol, 0, None)
    assert st == 2 and b"alias" in lib.fsyrk_b200_last_error()  # aliased output is rejected (test_fast_syrk.cpp:377-385)
    c = np.zeros((8, 8), dtype=np.uint64)
    st = lib.fsyrk_b200_syrk_fast_into(7, a.ctypes.data_as(u64p), 8, 8, 4, c.ctypes.data_as(u64p), 8, pol, 0, None)
    assert st == 1  # DimensionError
    st = lib.fsyrk_b200_syrk_fast_into(8, a.ctypes.data_as(u64p), 8, 8, 8, c.ctypes.data_as(u64p), 8, pol, 0, None)
    assert st == 2


def test_no_cpu_fallback(fsyrk):
    if fsyrk.device_available():
        pytest.skip("device present")
    f = fsyrk.PrimeField(131071)
    a = fsyrk.random_matrix(f, 16, 16, 1)
    with pytest.raises(fsyrk.DeviceError):
        fsyrk.syrk_fast(f, a, fsyrk.make_syrk_plan(f, fsyrk.RecursionPolicy(2)))


def test_python_mirror_shape_errors(fsyrk):
    f = fsyrk.PrimeField(7)
    plan = fsyrk.make_syrk_plan(f, fsyrk.RecursionPolicy(2))
    with pytest.raises(fsyrk.DimensionError):
        fsyrk.syrk_fast_into(f, np.zeros((4, 3), np.uint64), np.zeros((5, 5), np.uint64), plan)
    with pytest.raises(fsyrk.DimensionError):
        fsyrk.syrkd(f, np.zeros((2, 2), np.uint64), [1], plan)
    with pytest.raises(ValueError):
        fsyrk.syrkd(fsyrk.PrimeField(2), np.ones((2, 2), np.uint64), [1, 1], plan)


def test_python_mirror_rejects_reversed_or_overlapping_rows(fsyrk):
    # a[::-1] has a negative row stride; an as_strided overlap has stride < 8*cols: neither is a
    # (data, rows, cols, ld) view, so both are refused before any library call
    f = fsyrk.PrimeField(7)
    plan = fsyrk.make_syrk_plan(f, fsyrk.RecursionPolicy(2))
    a = np.ones((6, 4), np.uint64)
    with pytest.raises(fsyrk.DimensionError):
        fsyrk.syrk_fast(f, a[::-1], plan)
    c = np.zeros((6, 6), np.uint64)
    with pytest.raises(fsyrk.DimensionError):
        fsyrk.syrk_fast_into(f, a, c[::-1], plan)
    over = np.lib.stride_tricks.as_strided(np.zeros(40, np.uint64), shape=(6, 6), strides=(16, 8))
    with pytest.raises(fsyrk.DimensionError):
        fsyrk.syrk_fast_into(f, a, over, plan)
    a2 = np.ones((4, 3, 2), np.uint64)
    with pytest.raises(fsyrk.DimensionError):
        fsyrk.herk_fast(fsyrk.QuadExtField(7), a2[::-1], fsyrk.make_herk_plan(fsyrk.QuadExtField(7), fsyrk.RecursionPolicy(2)))


def test_workspace_bytes_host_only(fsyrk):
    # the plan's device workspace is reported without touching a device (layout dry run);
    # the low-memory schedule moves the top level's P4 / P3 (2 h^2 uint32) into C12
    U = fsyrk.UNLIMITED_LEVELS
    for (p, n, k, thr, lev) in ((131071, 4096, 4096, 1024, U), (131071, 32768, 1024, 2, 1), (65521, 8192, 2048, 2, 1)):
        pol = fsyrk.RecursionPolicy(thr, lev)
        wide = fsyrk.workspace_bytes(p, n, k, pol)
        low = fsyrk.workspace_bytes(p, n, k, pol, lowmem=True)
        h = n // 2
        assert wide["arena"] - low["arena"] == 2 * h * h * 4
        assert wide["host_call"] == wide["arena"] + n * k * 8 + n * n * 8
    # a root leaf has no top-level products: both schedules coincide
    pol = fsyrk.RecursionPolicy(2, 0)
    assert fsyrk.workspace_bytes(7, 64, 64, pol)["arena"] == fsyrk.workspace_bytes(7, 64, 64, pol, lowmem=True)["arena"]
