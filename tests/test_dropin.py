"""The C++ drop-in shim (include/fsyrk_b200/fsyrk.hpp) against the reference's
own templates in one binary (tests/cpp/test_dropin.cpp, built in the build
container from the reference headers)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "tests", "cpp", "_build", "test_dropin")


def test_dropin_binary_links_the_product_library():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/test_dropin not built (needs the reference headers)")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libfsyrk_b200.so" in out


@pytest.mark.gpu
def test_dropin_against_reference_templates(gpu):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/_build/test_dropin missing: build it in the build container (make -C tests/cpp)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
