"""Tile schedules of the persistent product launch (csrc/driver.cu: Plan::balance_tiles, the
dynamic claim ring in csrc/tc_modmm_kernel.cuh) against the C oracle.

The schedule is chosen once per process (FSYRK_B200_SCHED: balanced by default, dynamic,
strided), so each mode runs in its own interpreter.  The shapes give every CTA several tiles of
different K (multi-level plans over each digit scheme, a K-chunked long-K leaf, the accumulating
form), which is what a schedule can get wrong: a tile run twice, skipped, or run with another
tile's K-chunk bookkeeping.  Reference semantics: fast_syrk.hpp:135-157 (the tree),
matrix.hpp:144-160 (exact dot products at any K).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, %(repo)r)
sys.path.insert(0, %(tests)r)
import oracle_py as orc
import paper_2001_04109_b200 as fs

checked = 0
for p in (65521, 65537, 131071, 998244353, 2147483647):
    f = fs.PrimeField(p)
    for (n, k, thr, lev) in ((1536, 1024, 128, 3), (1280, 640, 64, 2), (2048, 512, 512, 1)):
        a = orc.random_matrix(p, n, k, n + k + p %% 97)
        c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(thr, lev)))
        assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, n, k, thr, lev)
        checked += 1
    # accumulating form over a two-level plan
    n, k = 1024, 768
    a = orc.random_matrix(p, n, k, 5)
    c0 = orc.random_matrix(p, n, n, 6)
    c = c0.copy()
    fs.syrk_fast_acc(f, 3 %% p, a, 5 %% p, c, fs.make_syrk_plan(f, fs.RecursionPolicy(128, 2)))
    assert orc.lower_equal(c, orc.syrk_classical(p, a, 3 %% p, 5 %% p, c0)), (p, "acc")
    checked += 1
# a leaf whose K is drained in chunks (above the int32 bound of the 31-bit schemes)
for p, k in ((2147483647, 14000), (1000000007, 17000)):
    f = fs.PrimeField(p)
    a = orc.random_matrix(p, 640, k, 11)
    c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(4096, 0)))
    assert orc.lower_equal(c, orc.syrk_classical(p, a)), (p, "long K")
    checked += 1
# the same plan twice in a row: the dynamic counters must be rearmed by the first launch
f = fs.PrimeField(131071)
a = orc.random_matrix(131071, 2048, 2048, 3)
want = orc.syrk_classical(131071, a)
for _ in range(3):
    c = fs.syrk_fast(f, a, fs.make_syrk_plan(f, fs.RecursionPolicy(256)))
    assert orc.lower_equal(c, want)
    checked += 1
print("sched ok", checked)
"""


@pytest.mark.parametrize("mode", ["dynamic", "strided", "balanced"])
def test_tile_schedules_match_oracle(gpu, mode):
    env = dict(os.environ)
    env["FSYRK_B200_SCHED"] = mode
    code = CHILD % {"repo": REPO, "tests": os.path.join(REPO, "tests")}
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "sched ok 25" in r.stdout, r.stdout[-2000:]
