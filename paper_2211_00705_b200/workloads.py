"""Seeded synthetic inputs for the five BASELINE.json configurations (C1-C5).

This module is the ONLY thing the CUDA path and the CPU oracle share: it builds host
arrays (rho, rho*u per cell) and the constant records (EOS constants as printed in
BASELINE.json / PAPER.md, scheme parameters) from a counter-based SplitMix64 generator.
It holds none of the method's arithmetic: no pressures, fluxes, thresholds or solves.

Recipe:
  u01(c, f, m, j): s = 22110705; s = splitmix64(s ^ x) for x in (c, f, m, j);
                   return (s >> 11) * 2**-53.       U[a,b] = a + (b - a) * u01.
  c = config 1..5, f = field (0 density, 1 velocity, 2 location), m = member, j = element.
"""
from __future__ import annotations

import numpy as np

SEED = 22110705
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# 293 K constants as printed in BASELINE.json configs[0] (vapour p = a_v^2 rho with
# a_v^2 = 1.352e5; liquid p = p_sat + a_l^2 (rho - 998), a_l = 1500, p_sat = 2339).
# tau <= 0 and rho_tilde <= 0 ask each side to derive them (Maxwell, reading R3);
# p_min = -9e6 Pa is reading R3.
EOS_293K = {"a_v2": 1.352e5, "a_l": 1500.0, "rho0": 998.0, "p0": 2339.0,
            "tau": 0.0, "p_min": -9.0e6, "rho_tilde": 0.0}

# scheme parameters: C_CFL 0.9 (BASELINE configs[0]), eps_split 2, eps_tiny 0.5 (R4),
# theta_{k+-1} 0.9 and tolerances 1e-3 / 1e-1, l_max 1e6, Newton per R14.
PARAMS = {"cfl": 0.9, "eps_split": 2.0, "eps_tiny": 0.5, "theta_nb": 0.9, "tol_nb": 1e-3,
          "tol_tiny": 1e-1, "dts_max_iter": 1_000_000, "newton_rtol": 1e-13, "newton_gtol": 1e-12,
          "newton_max_iter": 50, "armijo_max": 30, "mode": 0}
MODE_SPLIT, MODE_EXPLICIT = 0, 1


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def u01(c, f, m, j) -> np.ndarray:
    """Counter-based uniform in [0, 1): vectorised over broadcastable m, j."""
    m = np.asarray(m, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    s = np.full(np.broadcast(m, j).shape, SEED, dtype=np.uint64)
    s = splitmix64(s ^ np.uint64(c))
    s = splitmix64(s ^ np.uint64(f))
    s = splitmix64(s ^ m)
    s = splitmix64(s ^ j)
    return (s >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(a, b, c, f, m, j):
    return a + (b - a) * u01(c, f, m, j)


class Workload(dict):
    """dict with keys: name, eos, params, M, N, cap, x_left, x_right, rho, mom (M x cap),
    and run control (steps or t_end)."""


def _alloc(M, cap):
    return np.zeros((M, cap)), np.zeros((M, cap))


def c1(cap_slack: int = 8) -> Workload:
    """BASELINE configs[0]: N=200 on [0,1]; liquid (1000, 0) left of x=0.5, vapour (0.02, 0)."""
    N, M = 200, 1
    rho, mom = _alloc(M, N + cap_slack)
    rho[0, :100] = 1000.0
    rho[0, 100:N] = 0.02
    return Workload(name="C1", eos=dict(EOS_293K), params=dict(PARAMS), M=M, N=N, cap=N + cap_slack,
                    x_left=0.0, x_right=1.0, rho=rho, mom=mom, t_end=2e-4)


def c2(mode: int = MODE_SPLIT, cap_slack: int = 16) -> Workload:
    """BASELINE configs[1]: N=1000 on [-0.5,0.5]; rho=1000, u=-50 (x<0), +50 (x>0)."""
    N, M = 1000, 1
    rho, mom = _alloc(M, N + cap_slack)
    rho[0, :N] = 1000.0
    mom[0, :500] = 1000.0 * -50.0
    mom[0, 500:N] = 1000.0 * 50.0
    p = dict(PARAMS)
    p["mode"] = mode
    return Workload(name="C2" + ("-explicit" if mode else ""), eos=dict(EOS_293K), params=p, M=M, N=N,
                    cap=N + cap_slack, x_left=-0.5, x_right=0.5, rho=rho, mom=mom, t_end=5e-4)


def c3(M: int = 65536, N: int = 1024, members=None, cap_slack: int = 32) -> Workload:
    """BASELINE configs[2]: per member rho=U[998,1002], |u|=U[20,200], jump x=U[0.3,0.7];
    u = -|u| left of the jump edge, +|u| right of it (expansion -> cavitation)."""
    mem = np.arange(M, dtype=np.uint64) if members is None else np.asarray(members, dtype=np.uint64)
    Mx = len(mem)
    rho0 = uniform(998.0, 1002.0, 3, 0, mem, 0)
    speed = uniform(20.0, 200.0, 3, 1, mem, 0)
    xj = uniform(0.3, 0.7, 3, 2, mem, 0)
    edge = np.floor(xj * N + 0.5).astype(np.int64)
    rho, mom = _alloc(Mx, N + cap_slack)
    i = np.arange(N)[None, :]
    rho[:, :N] = rho0[:, None]
    u = np.where(i < edge[:, None], -speed[:, None], speed[:, None])
    mom[:, :N] = rho[:, :N] * u
    return Workload(name="C3", eos=dict(EOS_293K), params=dict(PARAMS), M=Mx, N=N, cap=N + cap_slack,
                    x_left=0.0, x_right=1.0, rho=rho, mom=mom, steps=2000, members=mem)


def c4(M: int = 16384, N: int = 4096, members=None, cap_slack: int = 64) -> Workload:
    """BASELINE configs[3]: vapour rho=U[0.015,0.03], u0=U[10,100]; u=+u0 for i<N/2, -u0 after
    (collision at the midpoint -> nucleation where the phase criterion fires)."""
    mem = np.arange(M, dtype=np.uint64) if members is None else np.asarray(members, dtype=np.uint64)
    Mx = len(mem)
    rho0 = uniform(0.015, 0.03, 4, 0, mem, 0)
    u0 = uniform(10.0, 100.0, 4, 1, mem, 0)
    rho, mom = _alloc(Mx, N + cap_slack)
    i = np.arange(N)[None, :]
    rho[:, :N] = rho0[:, None]
    u = np.where(i < N // 2, u0[:, None], -u0[:, None])
    mom[:, :N] = rho[:, :N] * u
    return Workload(name="C4", eos=dict(EOS_293K), params=dict(PARAMS), M=Mx, N=N, cap=N + cap_slack,
                    x_left=0.0, x_right=1.0, rho=rho, mom=mom, steps=2000, members=mem)


def c5_segments(n_cells: int = 1 << 27, seg: int = 4096, first_segment: int = 0, n_segments=None):
    """BASELINE configs[4]: per 4096-cell segment s: rho_s=U[999,1001], v_s=U[-150,150]."""
    total = (n_cells + seg - 1) // seg
    n_segments = total - first_segment if n_segments is None else n_segments
    s = np.arange(first_segment, first_segment + n_segments, dtype=np.uint64)
    return uniform(999.0, 1001.0, 5, 0, 0, s), uniform(-150.0, 150.0, 5, 1, 0, s)


def c5(n_cells: int = 1 << 27, seg: int = 4096, h: float = 1e-3, slack: int = 16) -> Workload:
    """BASELINE configs[4]: one grid of n_cells (default 2^27) on [0, n_cells h], h = 1e-3 m;
    per 4096-cell segment rho = U[999,1001], v = U[-150,150]; capacity n_cells (1 + 1/slack)."""
    rs, vs = c5_segments(n_cells, seg)
    cap = n_cells + n_cells // slack
    rho = np.zeros((1, cap))
    mom = np.zeros((1, cap))
    rho[0, :n_cells] = np.repeat(rs, seg)[:n_cells]
    mom[0, :n_cells] = (np.repeat(rs, seg) * np.repeat(vs, seg))[:n_cells]
    return Workload(name="C5", eos=dict(EOS_293K), params=dict(PARAMS), M=1, N=n_cells, cap=cap,
                    x_left=0.0, x_right=n_cells * h, rho=rho, mom=mom, steps=500)
