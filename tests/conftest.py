import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    """Parse a tests/golden fixture: '# citation' lines, then sections
    'image', 'conn4', 'conn8' of whitespace-separated integer rows."""
    sections, cur, cites = {}, None, []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            if line.startswith("#"):
                cites.append(line)
                continue
            if line in ("image", "conn4", "conn8"):
                cur = line
                sections[cur] = []
                continue
            sections[cur].append([int(v) for v in line.split()])
    out = {k: np.array(v, dtype=np.int64) for k, v in sections.items()}
    out["image"] = out["image"].astype(np.uint8)
    out["conn4"] = out["conn4"].astype(np.int32)
    out["conn8"] = out["conn8"].astype(np.int32)
    out["citation"] = "\n".join(cites)
    return out


def golden_names():
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".txt"))


@pytest.fixture(scope="session")
def cuda_available():
    import torch
    return torch.cuda.is_available()
