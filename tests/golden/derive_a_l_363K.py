"""Back-derivation of the 363.15 K liquid sound speed a_l (tests/golden/eos_363K.txt).

The paper takes its liquid constants from steam tables that are not printed, so
a_l is derived from what the paper does print for the cavitation test:
the created bubble width h_V = 2.701184e-5 m.  With the reading R18 creation
solve (App. B), the created width is (w_r - w_l) dt0 and the first large step is
dt0 = C_CFL h0 / (|u| + a_l) = 0.5 * 0.01 / (4 + a_l) (the liquid sound
speed bounds S_max).  rho0 follows from the printed rho_min through the corrected Tait law
rho_min = rho0 + (p_min - p0)/a_l^2 (R1).

Only the CPU oracle is called (oracle/), never the CUDA path.  Run:
    python tests/golden/derive_a_l_363K.py
which prints the root; tests/test_oracle_pins.py checks that it reproduces the committed value.
"""
from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))


def created_width(a_l: float) -> float:
    from oracle import oracle as O
    from paper_2211_00705_b200 import workloads as W
    from conftest import read_golden
    g = read_golden("eos_363K.txt")
    cav = read_golden("cavitation_363K.txt")
    a_v2 = g["k_boltzmann"] * g["T0"] / ((2 * g["m_H"] + g["m_O"]) / g["N_A"])
    rho0 = g["rho_min"] - (g["p_min"] - g["p0"]) / a_l ** 2
    eos = {"a_v2": a_v2, "a_l": a_l, "rho0": rho0, "p0": g["p0"], "tau": 0.0, "p_min": g["p_min"],
           "rho_tilde": 0.0}
    r = rho0 + (cav["p_init"] - g["p0"]) / a_l ** 2  # liquid at p_init
    c = O.creation_solve(eos, W.PARAMS, 1, r, -cav["u_init"], r, cav["u_init"])
    dt0 = 0.5 * 0.01 / (cav["u_init"] + a_l)
    return (c["w_r"] - c["w_l"]) * dt0


def derive() -> float:
    from scipy.optimize import brentq
    from conftest import read_golden
    h_v = read_golden("cavitation_363K.txt")["h_V"]
    return brentq(lambda a: created_width(a) - h_v, 1400.0, 1600.0, xtol=1e-10, rtol=1e-14)


if __name__ == "__main__":
    a = derive()
    print(f"a_l = {a:.10f} m/s (committed value: 1479.6589)")
