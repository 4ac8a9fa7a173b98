"""ctypes wrapper of the CPU oracle (oracle/eiso.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and the
cpu_baseline / ``--impl reference`` legs of ``bench.py``.  The product package
(``paper_2211_00705_b200``) never imports this module; the two paths meet only in the
seeded input arrays of ``paper_2211_00705_b200.workloads`` (which holds no method
arithmetic).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-Wall", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC"]

VAP, LIQ, SPIN = 0, 1, 2
MODE_SPLIT, MODE_EXPLICIT, MODE_LTS, MODE_NEWTON = 0, 1, 2, 3


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, f) for f in ("eiso.c", "lax.c")]
    deps = srcs + [os.path.join(HERE, f) for f in ("eiso.h", "lax.h")]
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(map(os.path.getmtime, deps)):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB_PATH, *srcs, "-lm"])
    return LIB_PATH


class Eos(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("a_v2", "a_l", "rho0", "p0", "tau", "p_min", "rho_tilde")]


class Params(C.Structure):
    _fields_ = [("cfl", C.c_double), ("eps_split", C.c_double), ("eps_tiny", C.c_double),
                ("theta_nb", C.c_double), ("tol_nb", C.c_double), ("tol_tiny", C.c_double),
                ("dts_max_iter", C.c_int64), ("newton_rtol", C.c_double), ("newton_gtol", C.c_double),
                ("newton_max_iter", C.c_int32), ("armijo_max", C.c_int32), ("mode", C.c_int32)]


class Thresholds(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("rho_min", "rho_tilde", "p_tilde", "tau", "a_v")]


class Iface(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("p_minus", "p_plus", "rho_minus", "rho_plus", "u_minus",
                                          "u_plus", "z", "w", "F0", "F1")] + \
               [("iters", C.c_int32), ("status", C.c_int32)]


class Creation(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("p_A", "p_B", "rho_A", "rho_B", "u_B", "z_l", "z_r", "w_l",
                                          "w_r", "Fl0", "Fl1", "Fr0", "Fr1")] + \
               [("iters", C.c_int32), ("status", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("steps", "cell_updates", "dts_iters", "iface_solves",
                                         "creations", "splits", "merges", "regions")] + \
               [(n, C.c_double) for n in ("t_min", "t_max", "dt_min", "dt_max")] + \
               [("decision_margin_warnings", C.c_int64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Interface(C.Structure):
    _fields_ = [("member", C.c_int64), ("edge", C.c_int64), ("x", C.c_double),
                ("left_phase", C.c_int32), ("right_phase", C.c_int32),
                ("w", C.c_double), ("z", C.c_double), ("p_vap", C.c_double), ("p_liq", C.c_double),
                ("solve_status", C.c_int32), ("reserved", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        d = C.c_double
        L.eiso_thresholds_of.argtypes = [P(Eos), P(Thresholds)]
        L.eiso_phase.argtypes = [P(Eos), d]
        L.eiso_pressure.argtypes = [P(Eos), C.c_int, d]
        L.eiso_pressure.restype = d
        L.eiso_gibbs.argtypes = [P(Eos), C.c_int, d]
        L.eiso_gibbs.restype = d
        L.eiso_wave_f.argtypes = [P(Eos), C.c_int, d, d]
        L.eiso_wave_f.restype = d
        L.eiso_hll.argtypes = [P(Eos), d, d, d, d, P(d)]
        L.eiso_single_phase_star.argtypes = [P(Eos), C.c_int, d, d, d, d, P(d)]
        L.eiso_creation_trigger.argtypes = [P(Eos), C.c_int, d, d, d, d]
        L.eiso_interface_solve.argtypes = [P(Eos), P(Params), d, d, d, d, P(Iface)]
        L.eiso_creation_solve.argtypes = [P(Eos), P(Params), C.c_int, d, d, d, d, P(Creation)]
        L.eiso_create.argtypes = [P(Eos), P(Params), C.c_int64, C.c_int64, C.c_int64, d, d, P(C.c_void_p)]
        L.eiso_set_state.argtypes = [C.c_void_p, P(d), P(d), P(d), P(C.c_int64), d]
        L.eiso_set_threads.argtypes = [C.c_void_p, C.c_int]
        L.eiso_step.argtypes = [C.c_void_p, C.c_int64, P(Stats)]
        L.eiso_run_to.argtypes = [C.c_void_p, d, C.c_int64, P(Stats)]
        L.eiso_get_state.argtypes = [C.c_void_p, P(d), P(d), P(d), P(C.c_uint8), P(C.c_int64), P(d)]
        L.eiso_interfaces.argtypes = [C.c_void_p, P(Interface), C.c_int64, P(C.c_int64)]
        L.eiso_member_status.argtypes = [C.c_void_p, P(C.c_int32)]
        L.eiso_member_stats.argtypes = [C.c_void_p, C.c_int64, P(Stats)]
        L.eiso_destroy.argtypes = [C.c_void_p]
        L.eiso_lax_riemann.argtypes = [d, P(d), P(d), d, P(d), P(d), P(d), P(C.c_int32)]
        L.eiso_lax_flux.argtypes = [d, P(d), P(d), P(d)]
        L.eiso_lax_run.argtypes = [C.c_void_p, P(d), P(d), P(d), P(d), C.c_void_p]
        _lib = L
    return _lib


def make_eos(d: dict) -> Eos:
    return Eos(*(float(d[k]) for k in ("a_v2", "a_l", "rho0", "p0", "tau", "p_min", "rho_tilde")))


def make_params(d: dict) -> Params:
    return Params(float(d["cfl"]), float(d["eps_split"]), float(d["eps_tiny"]), float(d["theta_nb"]),
                  float(d["tol_nb"]), float(d["tol_tiny"]), int(d["dts_max_iter"]), float(d["newton_rtol"]),
                  float(d["newton_gtol"]), int(d["newton_max_iter"]), int(d["armijo_max"]), int(d["mode"]))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def thresholds(eos: dict) -> dict:
    t = Thresholds()
    s = lib().eiso_thresholds_of(C.byref(make_eos(eos)), C.byref(t))
    if s:
        raise ValueError(f"eiso_thresholds_of status {s}")
    return {n: getattr(t, n) for n, _ in t._fields_}


def phase(eos, rho):
    return lib().eiso_phase(C.byref(make_eos(eos)), rho)


def pressure(eos, ph, rho):
    return lib().eiso_pressure(C.byref(make_eos(eos)), ph, rho)


def gibbs(eos, ph, p):
    return lib().eiso_gibbs(C.byref(make_eos(eos)), ph, p)


def wave_f(eos, ph, rs, rk):
    return lib().eiso_wave_f(C.byref(make_eos(eos)), ph, rs, rk)


def hll(eos, rl, ml, rr, mr):
    F = (C.c_double * 2)()
    s = lib().eiso_hll(C.byref(make_eos(eos)), rl, ml, rr, mr, F)
    if s:
        raise ValueError(s)
    return F[0], F[1]


def single_phase_star(eos, ph, rl, ul, rr, ur):
    r = C.c_double()
    s = lib().eiso_single_phase_star(C.byref(make_eos(eos)), ph, rl, ul, rr, ur, C.byref(r))
    if s:
        raise ValueError(s)
    return r.value


def creation_trigger(eos, ph, rl, ul, rr, ur):
    return bool(lib().eiso_creation_trigger(C.byref(make_eos(eos)), ph, rl, ul, rr, ur))


def interface_solve(eos, params, rm, um, rp, up) -> dict:
    o = Iface()
    s = lib().eiso_interface_solve(C.byref(make_eos(eos)), C.byref(make_params(params)), rm, um, rp, up, C.byref(o))
    if s:
        raise ValueError(f"interface_solve status {s}")
    return {n: getattr(o, n) for n, _ in o._fields_}


def creation_solve(eos, params, phase_outer, rl, ul, rr, ur) -> dict:
    o = Creation()
    s = lib().eiso_creation_solve(C.byref(make_eos(eos)), C.byref(make_params(params)), phase_outer,
                                  rl, ul, rr, ur, C.byref(o))
    if s:
        raise ValueError(f"creation_solve status {s}")
    return {n: getattr(o, n) for n, _ in o._fields_}


class Sim:
    """Oracle simulation context (eiso_create ... eiso_destroy), host arrays only."""

    def __init__(self, eos: dict, params: dict, n_members: int, n_cells: int, capacity: int,
                 x_left: float, x_right: float, threads: int = 1):
        self.M, self.N, self.cap = int(n_members), int(n_cells), int(capacity)
        self._ctx = C.c_void_p()
        self._eos = make_eos(eos)
        self._prm = make_params(params)
        s = lib().eiso_create(C.byref(self._eos), C.byref(self._prm), self.M, self.N, self.cap,
                              float(x_left), float(x_right), C.byref(self._ctx))
        if s:
            raise ValueError(f"eiso_create status {s}")
        self.set_threads(threads)

    def set_threads(self, n: int):
        """OpenMP threads: over members (M > 1) or over one member's cells and regions."""
        if lib().eiso_set_threads(self._ctx, int(n)):
            raise ValueError("eiso_set_threads")

    def __del__(self):
        if getattr(self, "_ctx", None) and self._ctx.value and _lib is not None:
            try:
                _lib.eiso_destroy(self._ctx)
            except Exception:  # interpreter shutdown
                pass
            self._ctx = C.c_void_p()

    def set_state(self, rho, mom, width=None, n_cells=None, t0=0.0):
        rho = np.ascontiguousarray(rho, dtype=np.float64).reshape(self.M, self.cap)
        mom = np.ascontiguousarray(mom, dtype=np.float64).reshape(self.M, self.cap)
        w = None if width is None else np.ascontiguousarray(width, dtype=np.float64).reshape(self.M, self.cap)
        nc = None if n_cells is None else np.ascontiguousarray(n_cells, dtype=np.int64)
        s = lib().eiso_set_state(self._ctx, _dp(rho), _dp(mom), None if w is None else _dp(w),
                                 None if nc is None else nc.ctypes.data_as(C.POINTER(C.c_int64)), float(t0))
        if s:
            raise ValueError(f"eiso_set_state status {s}")

    def step(self, n_steps: int) -> dict:
        st = Stats()
        lib().eiso_step(self._ctx, int(n_steps), C.byref(st))
        return st.as_dict()

    def run_to(self, t_end: float, max_steps: int = 10 ** 9) -> dict:
        st = Stats()
        lib().eiso_run_to(self._ctx, float(t_end), int(max_steps), C.byref(st))
        return st.as_dict()

    def get_state(self):
        rho = np.zeros((self.M, self.cap))
        mom = np.zeros((self.M, self.cap))
        h = np.zeros((self.M, self.cap))
        ph = np.zeros((self.M, self.cap), dtype=np.uint8)
        n = np.zeros(self.M, dtype=np.int64)
        t = np.zeros(self.M)
        lib().eiso_get_state(self._ctx, _dp(rho), _dp(mom), _dp(h), ph.ctypes.data_as(C.POINTER(C.c_uint8)),
                             n.ctypes.data_as(C.POINTER(C.c_int64)), _dp(t))
        return {"rho": rho, "mom": mom, "h": h, "phase": ph, "n": n, "t": t}

    def interfaces(self):
        cnt = C.c_int64()
        lib().eiso_interfaces(self._ctx, None, 0, C.byref(cnt))
        arr = (Interface * max(cnt.value, 1))()
        lib().eiso_interfaces(self._ctx, arr, cnt.value, C.byref(cnt))
        return [{"member": a.member, "edge": a.edge, "x": a.x, "left_phase": a.left_phase,
                 "right_phase": a.right_phase, "w": a.w, "z": a.z, "p_vap": a.p_vap, "p_liq": a.p_liq,
                 "solve_status": a.solve_status} for a in arr[:cnt.value]]

    def member_status(self):
        out = np.zeros(self.M, dtype=np.int32)
        lib().eiso_member_status(self._ctx, out.ctypes.data_as(C.POINTER(C.c_int32)))
        return out

    def member_stats(self, m: int) -> dict:
        st = Stats()
        lib().eiso_member_stats(self._ctx, int(m), C.byref(st))
        return st.as_dict()


# ---------------- Lax shock tube (oracle/lax.c) ----------------

class LaxCase(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("gamma", "rho_l", "u_l", "p_l", "rho_r", "u_r", "p_r", "x_left",
                                          "x_right")] + \
               [("n", C.c_int64)] + [(n, C.c_double) for n in ("alpha", "theta_nb", "cfl", "t_end", "tol_nb",
                                                                "tol_tiny")] + \
               [("dts_max_iter", C.c_int64), ("implicit_block", C.c_int32)]


class LaxStats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("dts_iters", C.c_int64), ("dts_max", C.c_int64),
                ("riemann_solves", C.c_int64), ("t", C.c_double), ("status", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


LAX_DEFAULT = dict(gamma=1.4, rho_l=0.445, u_l=0.698, p_l=3.528, rho_r=0.5, u_r=0.0, p_r=0.571,
                   x_left=-5.0, x_right=5.0, n=100, alpha=1e-2, theta_nb=0.9, cfl=0.8, t_end=1.0,
                   tol_nb=1e-3, tol_tiny=1e-1, dts_max_iter=10 ** 8, implicit_block=1)


def lax_case(**kw) -> LaxCase:
    d = dict(LAX_DEFAULT)
    d.update(kw)
    return LaxCase(**d)


def lax_riemann(gamma, wl, wr, xi=0.0):
    """Exact gamma-law Riemann solution sampled at x/t = xi: (prim (rho,u,p), p*, u*, iters)."""
    a = (C.c_double * 3)(*wl)
    b = (C.c_double * 3)(*wr)
    out = (C.c_double * 3)()
    ps, us, it = C.c_double(), C.c_double(), C.c_int32()
    s = lib().eiso_lax_riemann(C.c_double(gamma), a, b, C.c_double(xi), out, C.byref(ps), C.byref(us), C.byref(it))
    if s:
        raise ValueError(f"eiso_lax_riemann status {s}")
    return np.array(out[:]), ps.value, us.value, it.value


def lax_run(case: LaxCase):
    """Runs one Lax case; returns (rho, mom, E, x_faces, stats dict)."""
    nc = case.n + 1
    rho, mom, E = np.zeros(nc), np.zeros(nc), np.zeros(nc)
    xf = np.zeros(nc + 1)
    st = LaxStats()
    lib().eiso_lax_run(C.byref(case), _dp(rho), _dp(mom), _dp(E), _dp(xf), C.byref(st))
    return rho, mom, E, xf, st.as_dict()
