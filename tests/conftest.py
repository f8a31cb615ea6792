import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def h2mech():
    from workload import load_mech
    return load_mech("h2_9sp")


@pytest.fixture(scope="session")
def ch4mech():
    from workload import load_mech
    return load_mech("ch4_20sp")


def synth_mech(ns, W, nasa=None, visc=None, cond=None, diff=None, Tmid=1000.0):
    """A synthetic mechanism: species k is made of one atom of its own element
    of atomic weight W[k] (so W_k = W[k] exactly).  NASA/transport coefficients
    default to zero except a1 = 3.5."""
    W = np.asarray(W, dtype=np.float64)
    lo = np.zeros((ns, 7)); lo[:, 0] = 3.5
    if nasa is not None:
        lo = np.asarray(nasa, dtype=np.float64).reshape(ns, 7)
    npair = ns * (ns + 1) // 2
    return {
        "name": "synthetic", "species": [f"S{k}" for k in range(ns)], "elements": [f"E{k}" for k in range(ns)],
        "ns": ns, "ne": ns, "W_elem": W.copy(), "atoms": np.eye(ns, dtype=np.int32),
        "nasa_lo": lo.copy(), "nasa_hi": lo.copy(),
        "T_lo": np.full(ns, 200.0), "T_mid": np.full(ns, Tmid), "T_hi": np.full(ns, 3500.0),
        "visc": np.zeros((ns, 5)) if visc is None else np.asarray(visc, dtype=np.float64),
        "cond": np.zeros((ns, 5)) if cond is None else np.asarray(cond, dtype=np.float64),
        "diff": np.zeros((npair, 5)) if diff is None else np.asarray(diff, dtype=np.float64),
        "inert": np.zeros(ns, dtype=np.uint8),
    }
