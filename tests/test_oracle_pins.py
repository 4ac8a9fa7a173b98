"""Pins of the CPU oracle to values PRINTED IN THE PAPER (tests/golden/*, each with its
PAPER.md line).  These do not use the CUDA path.  A dropped term, sign or index in the EOS,
Gibbs energies, kinetic relation (reading R2), the two-phase / creation systems (App. A, B;
reading R18), the Maxwell construction (R3) or the CFL rule (R4-R6) moves at least one of
these printed digits."""
import math

import numpy as np
import pytest

from conftest import eos_363K, read_golden
from paper_2211_00705_b200 import workloads as W

LIQ, VAP = 1, 0


@pytest.fixture(scope="module")
def eos():
    return eos_363K()


def test_kT0_over_m_from_printed_constants(eos):
    # kT0/m with the printed k, m and T0 = 363.15 K
    assert eos["a_v2"] == pytest.approx(167601.3186896, rel=1e-12)


def test_maxwell_thresholds_363K(oracle_mod, eos):
    """P1: tab:max_vap_lintait363 from the equal-area rule along liquid -> linear
    spinodal -> vapour (reading R3)."""
    g = read_golden("thresholds_363K.txt")
    t = oracle_mod.thresholds(eos)
    assert t["p_tilde"] == pytest.approx(g["p_tilde"], abs=1e-6)
    assert t["rho_tilde"] == pytest.approx(g["rho_tilde"], abs=1e-6)
    assert t["rho_min"] == pytest.approx(965.289008, abs=1e-9)


def test_tau_formula_363K(oracle_mod, eos):
    # tau = (2 pi)^-1/2 (m/(k T0))^{3/2}
    t = oracle_mod.thresholds(eos)
    assert t["tau"] == pytest.approx((2 * math.pi) ** -0.5 * eos["a_v2"] ** -1.5, rel=1e-14)


def _liquid_density(eos, p):
    return eos["rho0"] + (p - eos["p0"]) / eos["a_l"] ** 2


def test_cavitation_star_state(oracle_mod, eos):
    """P2/P4: tab:sol_dat_4_p/u exact rows, w, h_V."""
    g = read_golden("cavitation_363K.txt")
    r = _liquid_density(eos, g["p_init"])
    c = oracle_mod.creation_solve(eos, W.PARAMS, LIQ, r, -g["u_init"], r, g["u_init"])
    assert c["p_A"] == pytest.approx(g["p_L_star"], abs=1e-6)
    assert c["p_B"] == pytest.approx(g["p_V_star"], abs=1e-6)
    assert abs(c["u_B"] - g["u_V_star"]) < 1e-12
    u_L_left = -g["u_init"] - oracle_mod.wave_f(eos, LIQ, c["rho_A"], r)
    assert u_L_left == pytest.approx(-g["u_L_star"], abs=1e-6)
    assert c["w_r"] == pytest.approx(g["w"], abs=1e-6)
    assert c["w_l"] == pytest.approx(-g["w"], abs=1e-6)
    # created width (w_r - w_l) dt0 with dt0 = C h0 / S_max (a_l was fitted from this number,
    # so this is a consistency check, not an independent pin)
    dt0 = 0.5 * 0.01 / (g["u_init"] + eos["a_l"])
    assert (c["w_r"] - c["w_l"]) * dt0 == pytest.approx(g["h_V"], abs=1e-12)


def test_nucleation_star_state(oracle_mod, eos):
    """P3: tab:sol_dat_3_p/u exact rows and w."""
    g = read_golden("nucleation_363K.txt")
    r = g["p_init"] / eos["a_v2"]
    c = oracle_mod.creation_solve(eos, W.PARAMS, VAP, r, g["u_init"], r, -g["u_init"])
    assert c["p_A"] == pytest.approx(g["p_V_star"], abs=1.5e-6)
    assert c["p_B"] == pytest.approx(g["p_L_star"], abs=1e-6)
    assert abs(c["u_B"] - g["u_L_star"]) < 1e-12
    u_V_left = g["u_init"] - oracle_mod.wave_f(eos, VAP, c["rho_A"], r)
    assert u_V_left == pytest.approx(g["u_V_star"], abs=1e-6)
    assert c["w_r"] == pytest.approx(g["w"], abs=1e-6)


_RUNS = {}


def _run_363K(oracle_mod, eos, kind, mode=0):
    """The paper's 363.15 K run (cached: the nucleation run takes seconds)."""
    if (kind, mode) not in _RUNS:
        _RUNS[(kind, mode)] = _run_363K_fresh(oracle_mod, eos, kind, mode)
    return _RUNS[(kind, mode)]


def _run_363K_fresh(oracle_mod, eos, kind, mode):
    g = read_golden("cavitation_363K.txt" if kind == "cav" else "nucleation_363K.txt")
    N, cap = 400, 416
    if kind == "cav":
        r = _liquid_density(eos, g["p_init"])
        uL = -g["u_init"]
    else:
        r = g["p_init"] / eos["a_v2"]
        uL = g["u_init"]
    prm = dict(W.PARAMS)
    prm["cfl"] = 0.5  # P:1233 / P:1367
    prm["mode"] = mode
    s = oracle_mod.Sim(eos, prm, 1, N, cap, -2.0, 2.0)  # h0 = 1e-2 on [-2, 2]
    rho = np.zeros((1, cap))
    mom = np.zeros((1, cap))
    rho[0, :N] = r
    mom[0, :N // 2] = r * uL
    mom[0, N // 2:N] = -r * uL
    s.set_state(rho, mom)
    st = s.run_to(5e-4)
    return g, s, st


def test_cavitation_run_166_steps(oracle_mod, eos):
    """P5: the CFL rule (R5: S_max over all cells; R6: h_min over non-tiny cells) and eps_tiny
    (R4) reproduce the printed 166 large steps; bubble width."""
    g, s, st = _run_363K(oracle_mod, eos, "cav")
    assert s.member_status()[0] == 0
    assert st["steps"] == int(g["large_steps"])
    assert st["creations"] == 1
    xs = [i["x"] for i in s.interfaces()]
    assert len(xs) == 2
    assert xs[1] - xs[0] == pytest.approx(g["bubble_width_t_end"], rel=1e-5)
    # star plateau next to the bubble approaches the exact star pressure (P:1277 explicit/implicit rows)
    st8 = s.get_state()
    k = int(np.argmin(st8["rho"][0, :st8["n"][0]]))  # the vapour cell
    p_vap = eos["a_v2"] * st8["rho"][0, k]
    assert p_vap == pytest.approx(g["p_V_star"], abs=0.05)


@pytest.mark.slow
def test_nucleation_run_droplet_width(oracle_mod, eos):
    """P:1422 droplet width (w_r - w_l) t_end = 2.03e-7 m and P:1424 ~143 large steps
    (reading R21 gives 146: soft)."""
    g, s, st = _run_363K(oracle_mod, eos, "nuc")
    assert s.member_status()[0] == 0
    xs = [i["x"] for i in s.interfaces()]
    assert xs[1] - xs[0] == pytest.approx(g["droplet_width_t_end"], rel=2e-2)
    assert abs(st["steps"] - g["large_steps"]) <= 4


def test_interface_report_cavitation_star_state(oracle_mod, eos):
    """eis_interfaces' Riemann report (App. A) at the end of the cavitation run: the bubble's
    adjacent cells hold the exact star states, so the reported star pressures and boundary
    speed are the paper's printed ones (P:1277 p_V*, p_L*; P:1264 w) to the printed digits."""
    g, s, st = _run_363K(oracle_mod, eos, "cav")
    ifc = s.interfaces()
    assert len(ifc) == 2 and all(i["solve_status"] == 0 for i in ifc)
    for i, sign in zip(ifc, (-1.0, 1.0)):
        assert i["p_vap"] == pytest.approx(g["p_V_star"], abs=1e-6)
        assert i["p_liq"] == pytest.approx(g["p_L_star"], abs=1e-6)
        assert i["w"] == pytest.approx(sign * g["w"], abs=1e-6)
        assert i["z"] * sign > 0  # evaporation: mass flows from the liquid into the bubble


def test_interface_report_nucleation(oracle_mod, eos):
    """The same report on the nucleation run: the droplet's boundary speed is the printed w
    (2.03e-4 m/s) and the star pressures agree with P:1390 within the scheme's
    smearing of the outer waves (1e-6 relative)."""
    g, s, st = _run_363K(oracle_mod, eos, "nuc")
    ifc = s.interfaces()
    assert len(ifc) == 2 and all(i["solve_status"] == 0 for i in ifc)
    for i, sign in zip(ifc, (-1.0, 1.0)):
        assert i["w"] == pytest.approx(sign * g["w"], rel=2e-2)
        assert i["p_vap"] == pytest.approx(g["p_V_star"], rel=1e-6)
        assert i["p_liq"] == pytest.approx(g["p_L_star"], rel=1e-6)


def test_cavitation_dts_local_iterations(oracle_mod, eos):
    """Alg. 2's stop rule and residual against the paper's count of local
    iterations for the cavitation test: 355 DTS iterations over the 166 large steps
    (tab:comp_costs_2); the oracle gives 335.  Mistakes in the loop move the total by
    more than 10 % (measured with this oracle: theta_nb 0.5 instead of 0.9 -> 429; tol_nb 1e-4
    instead of 1e-3 -> 405; the two tolerances swapped -> 286).  Every stop decision of this run
    is clear of its rounding floor (no decision-margin warning), so the count is a property of
    the method, not of the arithmetic."""
    g, s, st = _run_363K(oracle_mod, eos, "cav")
    assert st["steps"] == int(g["large_steps"])
    assert st["dts_iters"] == pytest.approx(g["dts_local_iterations"], rel=0.10)
    assert st["decision_margin_warnings"] == 0


@pytest.mark.slow
def test_nucleation_dts_local_iterations_rounding_regime(oracle_mod, eos):
    """The nucleation test's count (tab:comp_costs_3: 1,367,460 DTS iterations over 143
    steps) sits in the regime the paper warns about (with dtau_k ~ 6e-12 "only few
    meaningful digits" remain).  Pinned two ways (reading R28): the total is within a factor 3
    of the printed one, and the oracle's own decision-margin accounting flags the DTS stop of
    (nearly) every large step as lying within the rounding-error bound of its residual test,
    which is why no tighter agreement with the printed count can be expected from any fp64
    implementation."""
    g, s, st = _run_363K(oracle_mod, eos, "nuc")
    assert s.member_status()[0] == 0
    ratio = st["dts_iters"] / g["dts_local_iterations"]
    assert 1 / 3 <= ratio <= 3, ratio
    assert st["decision_margin_warnings"] >= 0.8 * st["regions"], (st["decision_margin_warnings"], st["regions"])


def test_a_l_363K_back_derivation_reproduces_the_committed_value():
    """tests/golden/derive_a_l_363K.py (oracle only) reproduces the committed a_l from the
    printed created width h_V."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "derive_a_l_363K", os.path.join(os.path.dirname(__file__), "golden", "derive_a_l_363K.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.derive() == pytest.approx(read_golden("eos_363K.txt")["a_l"], abs=5e-5)
