import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def load_cases(name):
    """Unpacks tests/golden/<name>.npz into a list of dicts."""
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    n = int(z["n"])
    cases = [dict() for _ in range(n)]
    for key in z.files:
        if key == "n":
            continue
        i, field = key.split("_", 1)
        v = z[key]
        cases[int(i)][field] = v.item() if v.ndim == 0 else v
    for c in cases:
        if "data_x256" in c:
            c["data"] = c["data_x256"].astype(np.float64) / 256.0
    return cases


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle.Oracle()


@pytest.fixture(scope="session")
def reference_lib():
    import oracle
    if not os.path.exists(oracle.REF_SO):
        try:
            oracle.build()
        except Exception:
            pass
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref (reference build) not available")
    return oracle.Reference()


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def sslic():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import paper_1806_08741_b200 as s
    s.lib()
    return s
