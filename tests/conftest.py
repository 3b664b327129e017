import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as d:
        return {k: d[k] for k in d.files}


@pytest.fixture(scope="session")
def oracle():
    import vc3_oracle

    vc3_oracle.build()
    return vc3_oracle


@pytest.fixture(scope="session")
def vc3b():
    """The product package, with its CUDA library required to be present."""
    import paper_2003_02633_b200 as pkg
    from paper_2003_02633_b200 import _native

    _native.load()
    return pkg


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda", 0)


LAYOUT_NAMES = ["17_18", "base_16_16", "16_17", "17_17", "wide_10_25"]


def layout_by_name(name):
    from paper_2003_02633_b200.layout import BitLayout, LAYOUT_16_17, LAYOUT_17_17, LAYOUT_17_18, LAYOUT_BASE_16_16

    return {
        "17_18": LAYOUT_17_18,
        "base_16_16": LAYOUT_BASE_16_16,
        "16_17": LAYOUT_16_17,
        "17_17": LAYOUT_17_17,
        "wide_10_25": BitLayout(0, 7, 22, 10, 25, 80),
    }[name]


def policy_by_code(code):
    from paper_2003_02633_b200.layout import PrecisionPolicy

    word = {"S": "single", "D": "double"}
    return PrecisionPolicy(word[code[0]], word[code[1]], word[code[2]])
