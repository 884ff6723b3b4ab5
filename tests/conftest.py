import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle_bindings import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle_bindings import RefLib

    try:
        return RefLib()
    except (FileNotFoundError, OSError) as e:  # reference not built here
        pytest.skip(f"oracle/_ref not available: {e}")


@pytest.fixture(scope="session")
def girih():
    """The product package; built on demand (fails loudly if the build fails)."""
    import importlib

    lib = os.path.join(ROOT, "paper_1510_04995_b200", "libgirih_gpu.so")
    if not os.path.exists(lib):
        import __graft_entry__

        __graft_entry__.build()
    pkg = importlib.import_module("paper_1510_04995_b200")
    pkg.load()
    return pkg
