import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.dirname(os.path.abspath(__file__))):
    if _p not in sys.path:
        sys.path.insert(0, _p)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    """Parse a tests/golden fixture: blocks '<TAG> d0 d1 ...' followed by numbers."""
    blocks, tag, dims, vals = {}, None, None, []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            parts = line.split()
            if parts[0].isalpha():
                if tag is not None:
                    blocks[tag] = np.array(vals, dtype=np.float64).reshape(dims)
                tag, dims, vals = parts[0], [int(p) for p in parts[1:]], []
            else:
                vals.extend(float(p) for p in parts)
    if tag is not None:
        blocks[tag] = np.array(vals, dtype=np.float64).reshape(dims)
    return blocks


@pytest.fixture
def golden():
    return load_golden
