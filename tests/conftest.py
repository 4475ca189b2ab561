import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def sim():
    from paper_2511_21669_b200 import Simulator
    s = Simulator(0)
    yield s
    s.close()


@pytest.fixture(scope="session")
def gen_dir():
    """Large fixtures (mixed.jsonl, model.json) regenerated through the reference oracle."""
    import reforacle
    reforacle.ensure_generated()
    return reforacle.GEN_DIR
