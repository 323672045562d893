import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def build_product():
    """Compile libgsmart.so (in-tree, sm_100a) without importing the package
    first (the package loads the library at import)."""
    import importlib.util
    path = os.path.join(ROOT, "paper_2106_14038_b200", "build.py")
    spec = importlib.util.spec_from_file_location("_gsmart_build", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden_fig():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "fig1_fig2.json")) as f:
        return json.load(f)
