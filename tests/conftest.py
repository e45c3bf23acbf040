import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long-running (large N)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def paper_tables():
    return json.loads((GOLDEN / "paper_tables.json").read_text())


@pytest.fixture(scope="session")
def baseline_ranks():
    p = GOLDEN / "baseline_ranks.json"
    return json.loads(p.read_text()) if p.exists() else []


@pytest.fixture(scope="session")
def hb():
    import paper_2209_05819_b200 as hb
    hb.load()
    return hb


@pytest.fixture(scope="session")
def ctx(hb):
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    c = hb.Context(0)
    yield c
    c.close()


def nthreads():
    return os.cpu_count() or 1
