import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    if name.endswith(".json"):
        return json.loads((GOLDEN / name).read_text())
    return np.load(GOLDEN / name, allow_pickle=True)


def unpack_states(g, prefix="train_"):
    """Site lists of the reference states stored by make_golden.pack_states."""
    chi, off, ent = g[prefix + "chi"], g[prefix + "site_off"], g[prefix + "entries"]
    out = []
    for n in range(chi.shape[0]):
        sites = []
        for s in range(chi.shape[1] - 1):
            size = chi[n, s] * 2 * chi[n, s + 1]
            sites.append(ent[off[n, s] : off[n, s] + size].reshape(chi[n, s], 2, chi[n, s + 1]))
        out.append(sites)
    return out


@pytest.fixture(scope="session")
def native():
    from paper_2411_09336_b200 import _native

    return _native.lib()
