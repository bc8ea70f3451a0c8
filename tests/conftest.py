import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def sp():
    from paper_2007_00056_b200 import sparsh
    return sparsh


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Port()


@pytest.fixture(scope="session")
def oracle_best():
    """The reference itself (oracle/_ref) when built, else the restatement."""
    import oracle
    return oracle.best_available()


@pytest.fixture(scope="session")
def ref():
    import oracle
    try:
        return oracle.Ref()
    except Exception:
        pytest.skip("oracle/_ref (reference build) not available")


def golden_path(name):
    return os.path.join(ROOT, "tests", "golden", name)


def experimental_built():
    """The library was built with SB_EXPERIMENTAL=1 (k_march, k_cross_rr, k_cross_tb2)."""
    try:
        from paper_2007_00056_b200 import _lib
        return bool(_lib.lib().sb_build_flags() & 1)
    except Exception:
        return False


needs_experimental = pytest.mark.skipif(not experimental_built(),
                                        reason="experimental kernels not built (make EXPERIMENTAL=1)")
