import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_cases.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA kernels through the C ABI)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


HYBRID_GOLDEN = ROOT / "tests" / "golden" / "hybrid_cases.npz"


@pytest.fixture(scope="session")
def hybrid_golden():
    with np.load(HYBRID_GOLDEN) as z:
        return {k: z[k] for k in z.files}


LASP1_GOLDEN = ROOT / "tests" / "golden" / "lasp1_cases.npz"


@pytest.fixture(scope="session")
def lasp1_golden():
    with np.load(LASP1_GOLDEN) as z:
        return {k: z[k] for k in z.files}
