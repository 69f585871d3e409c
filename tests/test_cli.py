"""The fsyrk_b200 CLI (tools/fsyrk_b200_cli.cpp) against the reference CLI's own checks
(proj/tests/cli_syrk_roundtrip.cmake), prime-field parts: file-based syrk, mirror, identity
scaling through syrkbd, the accumulating form, sos / nrsyf, and the exit codes."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "tools", "_build", "fsyrk_b200")


def run(*args):
    if not os.path.exists(CLI):
        subprocess.run(["make", "-C", os.path.join(REPO, "tools")], check=True, capture_output=True)
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=120)
    return r.returncode, r.stdout, r.stderr


def test_host_commands_and_exit_codes(tmp_path):
    # cli_syrk_roundtrip.cmake:24-25 and the usage errors (:33-36)
    assert run("sos", "--prime", 7, "--value", 6)[:2] == (0, "3 2\n")
    assert run("nrsyf", "--prime", 7, "--alpha", 3, "--beta", 5)[:2] == (0, "1 3\n1 2\n")
    assert run("verify", "--prime", 4)[0] == 2
    assert run("syrk", "--input", tmp_path / "does_not_exist.txt")[0] == 2
    assert run("count", "--n", 5)[0] == 2
    assert run("nope")[0] == 2
    assert run("syrk", "--field", "gf2k", "--input", tmp_path / "x")[0] == 2
    assert run("nrsyf", "--prime", 7, "--alpha", 2, "--beta", 5)[0] == 2  # 2 is a residue mod 7
    bad = tmp_path / "bad.txt"
    bad.write_text("2 2\n1 2\n3 101\n")  # 101 is not a residue mod 101
    rc, _, err = run("syrk", "--prime", 101, "--input", bad)
    assert rc == 2 and "invalid F_101 element" in err


@pytest.mark.gpu
def test_file_roundtrips(tmp_path):
    a = tmp_path / "cli_in.txt"
    a.write_text("2 2\n1 2\n3 4\n")
    assert run("syrk", "--field", "fp", "--prime", 101, "--input", a)[:2] == (0, "2 2\n5 0\n11 25\n")
    assert run("syrk", "--field", "fp", "--prime", 101, "--input", a, "--mirror")[:2] == (0, "2 2\n5 11\n11 25\n")
    sc = tmp_path / "cli_scale.txt"
    sc.write_text("S 1\nS 1\n")
    assert run("syrk", "--prime", 101, "--input", a, "--scaling", sc)[:2] == (0, "2 2\n5 0\n11 25\n")
    c0 = tmp_path / "cli_c0.txt"
    c0.write_text("2 2\n1 0\n0 1\n")
    assert run("syrk", "--prime", 101, "--input", a, "--alpha", 2, "--beta", 3, "--acc", c0)[:2] == \
        (0, "2 2\n13 0\n22 53\n")
    out = tmp_path / "c.txt"
    assert run("syrk", "--prime", 101, "--input", a, "--output", out)[0] == 0
    assert out.read_text() == "2 2\n5 0\n11 25\n"
    # antidiagonal block over F_7 (test_scaled_syrk.cpp:151-161)
    i2 = tmp_path / "i2.txt"
    i2.write_text("2 2\n1 0\n0 1\n")
    t = tmp_path / "t.txt"
    t.write_text("T 1 0\n")
    assert run("syrk", "--prime", 7, "--input", i2, "--scaling", t, "--mirror")[:2] == (0, "2 2\n0 1\n1 0\n")


@pytest.mark.gpu
def test_verify_and_bench():
    rc, out, _ = run("verify", "--field", "fp", "--prime", 131071, "--n", 48, "--cases", 10)
    assert rc == 0 and out.strip().endswith("PASS overall"), out
    # cli_syrk_roundtrip.cmake:29: the F_{p^2} battery (syrk_fast and herk_fast)
    rc, out, _ = run("verify", "--field", "fp2", "--prime", 13, "--n", 24, "--cases", 6)
    assert rc == 0 and "herk_fast" in out and out.strip().endswith("PASS overall"), out
    rc, out, _ = run("bench", "--prime", 131071, "--min-n", 256, "--max-n", 512, "--threshold", 128)
    lines = out.strip().splitlines()
    assert rc == 0 and lines[0] == "algorithm,n,seconds,effective_gfops" and len(lines) == 3


@pytest.mark.gpu
def test_fp2_file_syrk(tmp_path):
    import numpy as np
    import sys
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import oracle_py as orc
    p, n, k = 13, 5, 4
    a = orc.random_matrix(p, n, 2 * k, 9).reshape(n, k, 2)
    f = tmp_path / "a2.txt"
    f.write_text(f"{n} {k}\n" + "\n".join(" ".join(str(int(x[0] + x[1] * p)) for x in row) for row in a) + "\n")
    rc, out, err = run("syrk", "--field", "fp2", "--prime", p, "--input", f)
    assert rc == 0, err
    rows = [list(map(int, l.split())) for l in out.strip().splitlines()[1:]]
    want = orc.fp2_syrk_classical(p, a, False)
    for i in range(n):
        for j in range(n):
            enc = int(want[i, j, 0] + want[i, j, 1] * p) if j <= i else 0
            assert rows[i][j] == enc, (i, j)
