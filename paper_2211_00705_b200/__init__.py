"""paper_2211_00705_b200 — B200-native hot path of May & Thein's explicit-implicit domain
splitting (arXiv 2211.00705) for 1D isothermal liquid-vapour flow with phase transition.

This module is the thin Python binding of ``libeis.so`` (C ABI in ``include/eis.h``):
argument marshalling only.  Every step of the method runs in the CUDA kernels of the
library; there is no CPU fallback.  Importing works without a GPU (the library loads), but
any context call needs a CUDA device and fails loudly otherwise.

Names follow the C ABI: ``eis_create`` -> :class:`Context`, ``eis_set_state`` ->
:meth:`Context.set_state`, ``eis_step`` -> :meth:`Context.step`, ``eis_run_to`` ->
:meth:`Context.run_to`, ``eis_get_state`` -> :meth:`Context.get_state`,
``eis_interfaces`` -> :meth:`Context.interfaces`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EIS_LIB") or os.path.join(HERE, "libeis.so")  # EIS_LIB: a variant build (tools)

EIS_HOST, EIS_DEVICE = 0, 1
MODE_SPLIT, MODE_EXPLICIT, MODE_LTS, MODE_NEWTON = 0, 1, 2, 3
LAYOUT_AUTO, LAYOUT_RESIDENT, LAYOUT_TILED = 0, 1, 2
STATUS = {0: "OK", 1: "E_ARG", 2: "E_ORDER", 3: "E_NONPOS_DENSITY", 4: "E_SPINODAL", 5: "E_NEWTON",
          6: "E_CREATION", 7: "E_DTS_CAP", 8: "E_WIDTH", 9: "E_CAPACITY", 10: "E_CUDA", 11: "E_NCCL",
          12: "E_UNSUPPORTED", 13: "E_INTERNAL"}


class EisError(RuntimeError):
    pass


class Eos(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("a_v2", "a_l", "rho0", "p0", "tau", "p_min", "rho_tilde")]


class Params(C.Structure):
    _fields_ = [("cfl", C.c_double), ("eps_split", C.c_double), ("eps_tiny", C.c_double),
                ("theta_nb", C.c_double), ("tol_nb", C.c_double), ("tol_tiny", C.c_double),
                ("dts_max_iter", C.c_int64), ("newton_rtol", C.c_double), ("newton_gtol", C.c_double),
                ("newton_max_iter", C.c_int32), ("armijo_max", C.c_int32), ("mode", C.c_int32),
                ("reserved", C.c_int32)]


class Grid(C.Structure):
    _fields_ = [("n_members", C.c_int64), ("n_cells", C.c_int64), ("cell_capacity", C.c_int64),
                ("x_left", C.c_double), ("x_right", C.c_double), ("h_av", C.c_double), ("device", C.c_int32),
                ("threads", C.c_int32), ("layout", C.c_int32), ("tile_cells", C.c_int32),
                ("nbr_left", C.c_int32), ("nbr_right", C.c_int32), ("stream", C.c_void_p)]


class Interface(C.Structure):
    _fields_ = [("member", C.c_int64), ("edge", C.c_int64), ("x", C.c_double),
                ("left_phase", C.c_int32), ("right_phase", C.c_int32),
                ("w", C.c_double), ("z", C.c_double), ("p_vap", C.c_double), ("p_liq", C.c_double),
                ("solve_status", C.c_int32), ("reserved", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("steps", "cell_updates", "dts_iters", "iface_solves",
                                         "creations", "splits", "merges", "regions")] + \
               [(n, C.c_double) for n in ("t_min", "t_max", "dt_min", "dt_max")] + \
               [("dts_iter_max", C.c_int64), ("decision_margin_warnings", C.c_int64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Thresholds(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("rho_min", "rho_tilde", "p_tilde", "tau", "a_v")]


# exported symbols of libeis.so (checked by tests/test_abi.py against include/eis.h)
SYMBOLS = ("eis_thresholds_of", "eis_create", "eis_set_state", "eis_step", "eis_run_to", "eis_get_state",
           "eis_interfaces", "eis_member_status", "eis_member_stats", "eis_last_error", "eis_destroy",
           "eis_set_exchange_buffer", "eis_set_exchange_peers", "eis_step_local", "eis_step_finish",
           "eis_tile_info", "eis_window_prediction", "eis_set_timing",
           "eis_get_timing", "eis_window_diag", "eis_lax_run")
# exchange-buffer layout (include/eis.h EIS_XB_*)
HALO = 10
XB_REC = 3 * HALO + 1
XB_SEND_LEFT, XB_SEND_RIGHT, XB_RECV_LEFT, XB_RECV_RIGHT = 0, XB_REC, 2 * XB_REC, 3 * XB_REC
XB_DT = 4 * XB_REC
XB_DOUBLES = 4 * XB_REC + 2
XB_MAXRANKS = 8
XB_DOUBLES_PEER = XB_DOUBLES + 4 * XB_REC + 8 * XB_MAXRANKS  # peer mode (eis_set_exchange_peers)

_lib = None


def lib():
    """Load libeis.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EisError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P, d, i64, i32, vp = C.POINTER, C.c_double, C.c_int64, C.c_int32, C.c_void_p
        L.eis_thresholds_of.argtypes = [P(Eos), P(Thresholds)]
        L.eis_create.argtypes = [P(Eos), P(Params), P(Grid), P(vp)]
        L.eis_set_state.argtypes = [vp, vp, vp, vp, vp, i32, d]
        L.eis_step.argtypes = [vp, i64, P(Stats)]
        L.eis_run_to.argtypes = [vp, d, i64, P(Stats)]
        L.eis_get_state.argtypes = [vp, vp, vp, vp, vp, vp, vp, i32]
        L.eis_interfaces.argtypes = [vp, P(Interface), i64, P(i64)]
        L.eis_member_status.argtypes = [vp, P(i32)]
        L.eis_member_stats.argtypes = [vp, P(Stats)]
        L.eis_tile_info.argtypes = [vp, P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        if not hasattr(L, "eis_window_prediction") and os.environ.get("EIS_LIB"):  # an older dev variant (A/B runs)
            L.eis_window_prediction = L.eis_tile_info
        L.eis_window_prediction.argtypes = [vp, P(C.c_int64), P(C.c_int64), P(i32)]
        L.eis_window_diag.argtypes = [vp, P(C.c_int64), C.c_int64, P(C.c_int64)]
        L.eis_set_timing.argtypes = [vp, C.c_int32]
        L.eis_get_timing.argtypes = [vp, P(C.c_double), P(C.c_int64)]
        L.eis_last_error.argtypes = [vp]
        L.eis_last_error.restype = C.c_char_p
        L.eis_destroy.argtypes = [vp]
        L.eis_set_exchange_buffer.argtypes = [vp, vp]
        L.eis_set_exchange_peers.argtypes = [vp, vp, vp, P(vp), i32, i32]
        L.eis_step_local.argtypes = [vp, d]
        L.eis_step_finish.argtypes = [vp, d, i32]
        L.eis_lax_run.argtypes = [P(LaxCase), i64, i64, vp, vp, vp, P(LaxStats), vp]
        for s in SYMBOLS:
            if s not in ("eis_last_error", "eis_destroy"):
                getattr(L, s).restype = C.c_int
        L.eis_destroy.restype = None
        _lib = L
    return _lib


def make_eos(d: dict) -> Eos:
    return Eos(*(float(d[k]) for k in ("a_v2", "a_l", "rho0", "p0", "tau", "p_min", "rho_tilde")))


def make_params(d: dict) -> Params:
    return Params(float(d["cfl"]), float(d["eps_split"]), float(d["eps_tiny"]), float(d["theta_nb"]),
                  float(d["tol_nb"]), float(d["tol_tiny"]), int(d["dts_max_iter"]), float(d["newton_rtol"]),
                  float(d["newton_gtol"]), int(d["newton_max_iter"]), int(d["armijo_max"]), int(d["mode"]), 0)


def eis_thresholds_of(eos: dict) -> dict:
    t = Thresholds()
    s = lib().eis_thresholds_of(C.byref(make_eos(eos)), C.byref(t))
    if s:
        raise EisError(f"eis_thresholds_of: {STATUS.get(s, s)}")
    return {n: getattr(t, n) for n, _ in t._fields_}


class LaxCase(C.Structure):
    """eis_lax_case (include/eis.h): one Lax shock tube with a small cell."""
    _fields_ = [(n, C.c_double) for n in ("gamma", "rho_l", "u_l", "p_l", "rho_r", "u_r", "p_r", "x_left",
                                          "x_right")] + [("n", C.c_int64)] + \
               [(n, C.c_double) for n in ("alpha", "theta_nb", "cfl", "t_end", "tol_nb", "tol_tiny")] + \
               [("dts_max_iter", C.c_int64), ("implicit_block", C.c_int32), ("dts_loop", C.c_int32)]


class LaxStats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("dts_iters", C.c_int64), ("dts_max", C.c_int64),
                ("riemann_solves", C.c_int64), ("t", C.c_double), ("status", C.c_int32), ("margins", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# the paper's Lax setup and DTS stop rule
LAX_DEFAULT = dict(gamma=1.4, rho_l=0.445, u_l=0.698, p_l=3.528, rho_r=0.5, u_r=0.0, p_r=0.571, x_left=-5.0,
                   x_right=5.0, n=100, alpha=1e-2, theta_nb=0.9, cfl=0.8, t_end=1.0, tol_nb=1e-3, tol_tiny=1e-1,
                   dts_max_iter=10 ** 9, implicit_block=1, dts_loop=0)


def lax_run(cases, stream=None):
    """eis_lax_run: a batch of Lax cases (dicts overriding LAX_DEFAULT), one CTA each, on the
    current CUDA device.  Returns (rho, mom, E) as (n_cases, stride) device tensors (row c holds
    case c's n + 1 cells) and the per-case stats dicts."""
    import torch
    recs = []
    for kw in cases:
        d = dict(LAX_DEFAULT)
        d.update(kw)
        recs.append(LaxCase(**d))
    n = len(recs)
    stride = max(r.n for r in recs) + 2
    arr = (LaxCase * n)(*recs)
    st = (LaxStats * n)()
    dev = torch.device("cuda", torch.cuda.current_device())
    rho, mom, E = (torch.zeros((n, stride), dtype=torch.float64, device=dev) for _ in range(3))
    if stream is None:
        stream = torch.cuda.current_stream()
    sh = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    s = lib().eis_lax_run(arr, n, stride, C.c_void_p(rho.data_ptr()), C.c_void_p(mom.data_ptr()),
                          C.c_void_p(E.data_ptr()), st, C.c_void_p(sh))
    if s:
        raise EisError(f"eis_lax_run: {STATUS.get(s, s)}")
    return rho, mom, E, [x.as_dict() for x in st]


def _ptr(a):
    """Device (torch) or host (numpy) buffer -> (address, where)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):  # torch tensor
        return a.data_ptr(), (EIS_DEVICE if a.is_cuda else EIS_HOST)
    return a.ctypes.data, EIS_HOST


class Context:
    """eis_create / eis_destroy.  ``stream``: a cudaStream_t handle (int) or a torch stream."""

    def __init__(self, eos: dict, params: dict, n_members: int, n_cells: int, capacity: int,
                 x_left: float, x_right: float, device: int = 0, stream=None, threads: int = 0,
                 layout: int = 0, tile_cells: int = 0, nbr_left: bool = False, nbr_right: bool = False,
                 h_av: float = 0.0):
        if stream is not None and hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        self.M, self.N, self.cap = int(n_members), int(n_cells), int(capacity)
        self.device = int(device)
        self._grid = Grid(self.M, self.N, self.cap, float(x_left), float(x_right), float(h_av), self.device, int(threads),
                          int(layout), int(tile_cells), int(bool(nbr_left)), int(bool(nbr_right)),
                          C.c_void_p(stream) if stream else None)
        self._eos, self._prm = make_eos(eos), make_params(params)
        self._ctx = C.c_void_p()
        s = lib().eis_create(C.byref(self._eos), C.byref(self._prm), C.byref(self._grid), C.byref(self._ctx))
        if s:
            raise EisError(f"eis_create: {STATUS.get(s, s)}")

    def _check(self, s, what):
        if s:
            msg = lib().eis_last_error(self._ctx)
            raise EisError(f"{what}: {STATUS.get(s, s)} ({msg.decode() if msg else ''})")

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value and _lib is not None:
            try:
                _lib.eis_destroy(self._ctx)
            except Exception:  # interpreter shutdown
                pass
            self._ctx = C.c_void_p()

    __del__ = close

    def set_state(self, rho, mom, width=None, n_cells=None, t0: float = 0.0):
        """rho, mom (and width): n_members*capacity fp64, host (numpy) or device (torch)."""
        pr, where = _ptr(rho)
        pm, w2 = _ptr(mom)
        pw, w3 = _ptr(width)
        pn, w4 = _ptr(n_cells)
        if w2 != where or (w3 is not None and w3 != where) or (w4 is not None and w4 != where):
            raise EisError("set_state: all buffers must be host or all device")
        self._check(lib().eis_set_state(self._ctx, pr, pm, pw, pn, where, float(t0)), "eis_set_state")

    def step(self, n_steps: int, stats: bool = False):
        st = Stats()
        self._check(lib().eis_step(self._ctx, int(n_steps), C.byref(st) if stats else None), "eis_step")
        return st.as_dict() if stats else None

    def run_to(self, t_end: float, max_steps: int = 10 ** 9, stats: bool = False):
        st = Stats()
        self._check(lib().eis_run_to(self._ctx, float(t_end), int(max_steps), C.byref(st) if stats else None),
                    "eis_run_to")
        return st.as_dict() if stats else None

    def get_state(self, out: dict | None = None) -> dict:
        """Host copy (numpy) unless ``out`` holds device tensors (rho, mom, h, phase, n, t)."""
        if out is None:
            out = {"rho": np.zeros((self.M, self.cap)), "mom": np.zeros((self.M, self.cap)),
                   "h": np.zeros((self.M, self.cap)), "phase": np.zeros((self.M, self.cap), np.uint8),
                   "n": np.zeros(self.M, np.int64), "t": np.zeros(self.M)}
        ptrs = [_ptr(out.get(k)) for k in ("rho", "mom", "h", "phase", "n", "t")]
        where = next(w for _, w in ptrs if w is not None)
        self._check(lib().eis_get_state(self._ctx, *[p for p, _ in ptrs], where), "eis_get_state")
        return out

    def interfaces(self) -> list:
        cnt = C.c_int64()
        self._check(lib().eis_interfaces(self._ctx, None, 0, C.byref(cnt)), "eis_interfaces")
        arr = (Interface * max(cnt.value, 1))()
        self._check(lib().eis_interfaces(self._ctx, arr, cnt.value, C.byref(cnt)), "eis_interfaces")
        return [{"member": a.member, "edge": a.edge, "x": a.x, "left_phase": a.left_phase,
                 "right_phase": a.right_phase, "w": a.w, "z": a.z, "p_vap": a.p_vap, "p_liq": a.p_liq,
                 "solve_status": a.solve_status} for a in arr[:cnt.value]]

    def member_status(self) -> np.ndarray:
        out = np.zeros(self.M, dtype=np.int32)
        self._check(lib().eis_member_status(self._ctx, out.ctypes.data_as(C.POINTER(C.c_int32))),
                    "eis_member_status")
        return out

    # ---- rank mode (tiled grid cut over ranks) ------------------------------------------
    def set_exchange_buffer(self, xbuf):
        """xbuf: a device tensor of XB_DOUBLES float64 owned by the caller (kept alive by it)."""
        self._xbuf = xbuf
        self._check(lib().eis_set_exchange_buffer(self._ctx, xbuf.data_ptr()), "eis_set_exchange_buffer")

    def set_exchange_peers(self, left_ptr, right_ptr, all_ptrs, rank: int, world: int):
        """Peer mode: device addresses (ints) of the neighbours' exchange buffers (None at the
        domain ends) and of every rank's, each XB_DOUBLES_PEER float64 (this rank's own buffer,
        set with set_exchange_buffer, must be all_ptrs[rank])."""
        arr = (C.c_void_p * len(all_ptrs))(*[int(a) for a in all_ptrs])
        self._check(lib().eis_set_exchange_peers(self._ctx, C.c_void_p(left_ptr) if left_ptr else None,
                                                 C.c_void_p(right_ptr) if right_ptr else None, arr,
                                                 int(rank), int(world)), "eis_set_exchange_peers")

    def step_local(self, t_end: float = float("inf")):
        self._check(lib().eis_step_local(self._ctx, float(t_end)), "eis_step_local")

    def step_finish(self, t_end: float = float("inf"), after_step: bool = True):
        self._check(lib().eis_step_finish(self._ctx, float(t_end), int(bool(after_step))), "eis_step_finish")

    def window_diag(self):
        """(count, 11) int64: cycles, DTS iterations, window cells, boundaries, start clock, 6 phases."""
        n = C.c_int64()
        self._check(lib().eis_window_diag(self._ctx, None, 0, C.byref(n)), "eis_window_diag")
        out = np.zeros((max(n.value, 1), 11), dtype=np.int64)
        self._check(lib().eis_window_diag(self._ctx, out.ctypes.data_as(C.POINTER(C.c_int64)), n.value, C.byref(n)),
                    "eis_window_diag")
        return out[:n.value]

    def set_timing(self, enable: bool = True):
        self._check(lib().eis_set_timing(self._ctx, int(bool(enable))), "eis_set_timing")

    def get_timing(self) -> dict:
        ms = (C.c_double * 4)()
        n = C.c_int64()
        self._check(lib().eis_get_timing(self._ctx, ms, C.byref(n)), "eis_get_timing")
        return {"fast_ms": ms[0], "window_ms": ms[1], "tile_ms": ms[2], "resident_ms": ms[3], "launches": n.value}

    def tile_info(self) -> dict:
        nt, full, win = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(lib().eis_tile_info(self._ctx, C.byref(nt), C.byref(full), C.byref(win)), "eis_tile_info")
        return {"n_tiles": nt.value, "full_tile_steps": full.value, "window_steps": win.value}

    def window_prediction(self) -> dict:
        w, h, en = C.c_int64(), C.c_int64(), C.c_int32()
        self._check(lib().eis_window_prediction(self._ctx, C.byref(w), C.byref(h), C.byref(en)), "eis_window_prediction")
        return {"windows": w.value, "predicted": h.value, "enabled": bool(en.value)}

    def member_stats(self) -> list:
        arr = (Stats * self.M)()
        self._check(lib().eis_member_stats(self._ctx, arr), "eis_member_stats")
        return [a.as_dict() for a in arr]
