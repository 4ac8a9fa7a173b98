import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_golden(name: str) -> dict:
    """Parse tests/golden/<name>: 'key = value  # citation' lines."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, v = (s.strip() for s in line.split("=", 1))
            out[k] = float(v)
    return out


def eos_363K() -> dict:
    g = read_golden("eos_363K.txt")
    a_v2 = g["k_boltzmann"] * g["T0"] / ((2 * g["m_H"] + g["m_O"]) / g["N_A"])
    rho0 = g["rho_min"] - (g["p_min"] - g["p0"]) / g["a_l"] ** 2
    return {"a_v2": a_v2, "a_l": g["a_l"], "rho0": rho0, "p0": g["p0"], "tau": 0.0,
            "p_min": g["p_min"], "rho_tilde": 0.0}


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    O.build()
    return O
