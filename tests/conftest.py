import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")
    # libcr.so (nvcc cross-compiles without a GPU) and the oracle's liboracle.so (g++)
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_cr_build", os.path.join(ROOT, "paper_2005_12692_b200", "build.py"))
    _b = importlib.util.module_from_spec(spec)  # not via the package: it refuses to import
    spec.loader.exec_module(_b)                 # without libcr.so
    _b.build()
    import oracle
    oracle.build()


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
