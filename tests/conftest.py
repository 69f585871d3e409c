import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running full-size parity case")


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(REPO, "tests", "golden", "reference_cases.npz")
    data = np.load(path, allow_pickle=False)
    cases = []
    for i in range(int(data["ncases"])):
        pre = f"c{i:03d}_"
        meta = data[pre + "meta"]
        rec = {
            "p": int(meta[0]), "n": int(meta[1]), "k": int(meta[2]), "seed": int(meta[3]),
            "threshold": int(meta[4]), "levels": None if int(meta[5]) < 0 else int(meta[5]),
            "mirror": bool(meta[6]), "alpha": int(meta[7]), "beta": int(meta[8]),
            "mode": str(data[pre + "mode"]), "A": data[pre + "A"], "C": data[pre + "C"],
            "digest": str(data[pre + "digest"]),
        }
        if pre + "C0" in data:
            rec["C0"] = data[pre + "C0"]
        if pre + "D" in data:
            rec["D"] = data[pre + "D"]
        if pre + "ns" in data:
            rec["ns"] = int(data[pre + "ns"])
        cases.append(rec)
    return {"cases": cases, "skew_p": data["skew_p"], "skew_form": data["skew_form"],
            "skew_a": data["skew_a"], "skew_b": data["skew_b"]}


@pytest.fixture(scope="session")
def fsyrk():
    import paper_2001_04109_b200 as m
    from paper_2001_04109_b200 import build
    build.build(verbose=False)
    return m


@pytest.fixture(scope="session")
def gpu(fsyrk):
    if not fsyrk.device_available():
        pytest.fail("gpu test on a machine without a usable sm_100 device")
    return fsyrk
