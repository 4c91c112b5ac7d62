import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    from oracle import pyoracle
    if not pyoracle.available("c"):
        pyoracle.build("c")
    lib = os.path.join(ROOT, "paper_2605_22014_b200", "libreshard_b200.so")
    if not os.path.exists(lib):
        import subprocess
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2605_22014_b200", "csrc")],
                       check=True)


_ensure_built()


@pytest.fixture(scope="session")
def oracle_c():
    from oracle.pyoracle import Oracle
    return Oracle("c")


@pytest.fixture(scope="session")
def oracle_ref():
    from oracle.pyoracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def golden():
    import json
    g = os.path.join(ROOT, "tests", "golden")
    out = {}
    for name in ("kat", "random_pairs", "baseline_plans", "c1_exec"):
        with open(os.path.join(g, name + ".json")) as f:
            out[name] = json.load(f)
    return out
