import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); the parity tests proper")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


@pytest.fixture(scope="session")
def golden():
    from tests.helpers import load_golden
    return load_golden()


def pytest_sessionstart(session):
    # (Re)build the in-tree sm_100a extension and the CPU oracle if stale.
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_pcd_build", os.path.join(ROOT, "paper_2406_01939_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True,
                   stdout=subprocess.DEVNULL)
