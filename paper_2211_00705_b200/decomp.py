"""One tiled grid cut over ranks (BASELINE configs[4] on several GPUs): tile-aligned slices, a
per-step halo exchange with the neighbour ranks and a min-reduction of the CFL pair.

Plumbing only: every step of the method runs in libeis kernels; this module
moves 10-cell halo records between ranks with torch.distributed (NCCL on GPUs, gloo on CPU)
and folds the (-S_max, h_min) pairs with an all-reduce(MIN).  Slices are whole tiles, so a
P-rank run computes exactly what the 1-rank run computes (min/max are exact, halos copy bits).
"""
from __future__ import annotations

import math

import torch

from . import (HALO, LAYOUT_TILED, XB_DOUBLES, XB_DOUBLES_PEER, XB_DT, XB_MAXRANKS, XB_REC, XB_RECV_LEFT,
               XB_RECV_RIGHT, XB_SEND_LEFT, XB_SEND_RIGHT, Context)


def tile_count(n: int, tile: int) -> int:
    """Tiles of the library's fixed-size tiling (the last takes the remainder, >= HALO cells)."""
    nt = max(1, math.ceil(n / tile))
    if nt > 1 and n - (nt - 1) * tile < HALO:
        nt -= 1
    return nt


def rank_slice(n: int, tile: int, rank: int, world: int) -> tuple[int, int]:
    """Cells [c0, c1) of rank `rank`: a contiguous, balanced range of whole tiles."""
    T = tile_count(n, tile)
    if T < world:
        raise ValueError(f"{T} tiles cannot be split over {world} ranks")
    t0, t1 = rank * T // world, (rank + 1) * T // world
    return t0 * tile, (n if rank == world - 1 else t1 * tile)


def exchange_halos(xbuf: torch.Tensor, rank: int, world: int, group=None) -> None:
    """send_left -> left rank's recv_right, send_right -> right rank's recv_left, then
    all-reduce(MIN) of the CFL pair.  Works for CUDA (NCCL) and CPU (gloo) tensors."""
    import torch.distributed as dist
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, xbuf[XB_SEND_LEFT:XB_SEND_LEFT + XB_REC], rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, xbuf[XB_RECV_LEFT:XB_RECV_LEFT + XB_REC], rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, xbuf[XB_SEND_RIGHT:XB_SEND_RIGHT + XB_REC], rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, xbuf[XB_RECV_RIGHT:XB_RECV_RIGHT + XB_REC], rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if world > 1:
        dist.all_reduce(xbuf[XB_DT:XB_DT + 2], op=dist.ReduceOp.MIN, group=group)


def capture_steps(step_once, k: int, stream):
    """A CUDA graph of k calls of step_once() captured on `stream` (a torch.cuda.Stream, the
    stream the library's contexts were created with): every call must only enqueue work on it
    (library steps, torch device ops, NCCL collectives).  Replaying it runs k whole steps with no
    host round trip between the per-step launches."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(k):
            step_once()
    return g


class StepGraphs:
    """Steps of a rank-mode grid as CUDA-graph replays: `graph_steps` steps per graph, captured
    once per t_end (the launch arguments are part of the graph); a remainder runs eagerly."""

    def __init__(self, step_once, stream, graph_steps: int):
        self.step_once, self.stream, self.k = step_once, stream, graph_steps
        self.graphs = {}

    def run(self, n_steps: int, t_end: float):
        g = self.graphs.get(t_end)
        if g is None and n_steps >= self.k:
            g = self.graphs[t_end] = capture_steps(lambda: self.step_once(t_end), self.k, self.stream)
        while g is not None and n_steps >= self.k:
            g.replay()
            n_steps -= self.k
        for _ in range(n_steps):
            self.step_once(t_end)


class RankGrid:
    """This rank's slice of one tiled grid.  For world == 1 it is a plain tiled context.

    graph_steps > 0 (world > 1): the per-step sequence step_local -> exchange -> step_finish is
    captured into a CUDA graph of graph_steps steps on a stream of the grid's own and replayed,
    so the host issues one replay per graph_steps steps instead of four calls per step.
    The first step (eager) initialises the NCCL communicators before any capture."""

    def __init__(self, eos: dict, params: dict, n_global: int, x_left: float, x_right: float, rank: int,
                 world: int, tile: int = 1400, device: int = 0, stream=None, group=None, slack: int = 16,
                 graph_steps: int = 0, peer: bool = False):
        self.rank, self.world, self.group = rank, world, group
        self.graph_steps = graph_steps if world > 1 else 0
        if self.graph_steps and (stream is None or stream == torch.cuda.default_stream(device)):
            stream = torch.cuda.Stream(device)  # capture needs a stream other than the default one
        self.stream = stream
        self._graphs = None
        self.c0, self.c1 = rank_slice(n_global, tile, rank, world)
        self.n = self.c1 - self.c0
        self.h_av = (x_right - x_left) / n_global
        self.cap = self.n + self.n // slack + tile
        self.ctx = Context(eos, params, 1, self.n, self.cap, x_left + self.c0 * self.h_av,
                           x_left + self.c1 * self.h_av, device=device, stream=stream, layout=LAYOUT_TILED,
                           tile_cells=tile, nbr_left=rank > 0, nbr_right=rank < world - 1, h_av=self.h_av)
        self.xbuf = None
        self.peer = False
        if world > 1:
            if peer:
                self.peer = self._setup_peers(device)
            if not self.peer:
                self.xbuf = torch.zeros(XB_DOUBLES, dtype=torch.float64, device=f"cuda:{device}")
                self.ctx.set_exchange_buffer(self.xbuf)

    def _setup_peers(self, device) -> bool:
        """Peer mode over torch symmetric memory (NVLink-mapped buffers of every rank): the
        kernels write the halo records and the CFL pair into the peers' buffers themselves and
        eis_step_finish waits for them -- no collective per step.  False (NCCL exchange) when
        symmetric memory is unavailable."""
        if self.world > XB_MAXRANKS:
            return False
        try:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(XB_DOUBLES_PEER, dtype=torch.float64, device=f"cuda:{device}")
            buf.zero_()
            hdl = symm_mem.rendezvous(buf, self.group if self.group is not None else dist.group.WORLD)
            ptrs = [int(p_) for p_ in hdl.buffer_ptrs]
            torch.cuda.synchronize(device)
            dist.barrier(group=self.group)  # every buffer zeroed before any rank publishes
        except Exception as exc:  # noqa: BLE001 -- no symmetric memory: the NCCL exchange
            import warnings
            warnings.warn(f"peer exchange unavailable ({exc}); using the NCCL exchange")
            return False
        self.xbuf, self._hdl = buf, hdl
        self.ctx.set_exchange_buffer(buf)
        r = self.rank
        self.ctx.set_exchange_peers(ptrs[r - 1] if r > 0 else None, ptrs[r + 1] if r < self.world - 1 else None,
                                    ptrs, r, self.world)
        return True

    def _on_stream(self):
        """torch's current stream = the library's stream (NCCL and torch ops ordered with the kernels)"""
        import contextlib
        return torch.cuda.stream(self.stream) if hasattr(self.stream, "cuda_stream") else contextlib.nullcontext()

    def exchange(self):
        if self.peer:  # the kernels exchanged over peer memory; eis_step_finish consumes it
            return
        with self._on_stream():
            exchange_halos(self.xbuf, self.rank, self.world, self.group)

    def set_state(self, rho_local, mom_local, t_end: float = float("inf")):
        """rho/mom: this rank's cells [c0, c1) (padded to cap), device or host buffers."""
        with self._on_stream():
            self.ctx.set_state(rho_local, mom_local)
            if self.world > 1:
                self.exchange()
                self.ctx.step_finish(t_end, after_step=False)

    def _step_once(self, t_end: float):
        self.ctx.step_local(t_end)
        self.exchange()
        self.ctx.step_finish(t_end, after_step=True)

    def step(self, n_steps: int, t_end: float = float("inf"), graph: bool = True):
        """graph=False: eager steps even when graph_steps > 0 (e.g. for per-kernel timing)."""
        if self.world == 1:
            return self.ctx.step(n_steps) if t_end == float("inf") else self.ctx.run_to(t_end, n_steps)
        with self._on_stream():
            if graph and self.graph_steps and n_steps > 0:
                if self._graphs is None:
                    self._step_once(t_end)  # eager: communicators and lazy module loads before capture
                    n_steps -= 1
                    self._graphs = StepGraphs(self._step_once, self.stream, self.graph_steps)
                self._graphs.run(n_steps, t_end)
                return
            for _ in range(n_steps):
                self._step_once(t_end)


class VirtualRanks:
    """P rank slices of one grid on ONE device, exchanged by device copies (no NCCL, no kernel
    waits on another): exercises the rank-mode library path against the 1-rank run."""

    def __init__(self, eos, params, n_global, x_left, x_right, world, tile=1400, device=0, stream=None,
                 peer: bool = False):
        """peer=True: the slices exchange through eis_set_exchange_peers (the kernels write into
        the neighbours' buffers, eis_step_finish consumes) instead of device copies; every rank's
        step_local is enqueued before any step_finish, so no kernel waits on a later one."""
        self.stream = stream
        self.peer = peer
        self._graphs = None
        self.parts = []
        for r in range(world):
            g = RankGrid.__new__(RankGrid)
            g.rank, g.world, g.group = r, world, None
            g.c0, g.c1 = rank_slice(n_global, tile, r, world)
            g.n = g.c1 - g.c0
            g.h_av = (x_right - x_left) / n_global
            g.cap = g.n + g.n // 16 + tile
            g.ctx = Context(eos, params, 1, g.n, g.cap, x_left + g.c0 * g.h_av, x_left + g.c1 * g.h_av,
                            device=device, stream=stream, layout=LAYOUT_TILED, tile_cells=tile,
                            nbr_left=r > 0, nbr_right=r < world - 1, h_av=g.h_av)
            g.xbuf = torch.zeros(XB_DOUBLES_PEER if peer else XB_DOUBLES, dtype=torch.float64, device=f"cuda:{device}")
            g.ctx.set_exchange_buffer(g.xbuf)
            self.parts.append(g)
        if peer:
            ptrs = [g.xbuf.data_ptr() for g in self.parts]
            for r, g in enumerate(self.parts):
                g.ctx.set_exchange_peers(ptrs[r - 1] if r > 0 else None, ptrs[r + 1] if r < world - 1 else None,
                                         ptrs, r, world)

    def _exchange(self):
        if self.peer:
            return
        P = self.parts
        for r, g in enumerate(P):
            if r > 0:
                g.xbuf[XB_RECV_LEFT:XB_RECV_LEFT + XB_REC].copy_(P[r - 1].xbuf[XB_SEND_RIGHT:XB_SEND_RIGHT + XB_REC])
            if r < len(P) - 1:
                g.xbuf[XB_RECV_RIGHT:XB_RECV_RIGHT + XB_REC].copy_(P[r + 1].xbuf[XB_SEND_LEFT:XB_SEND_LEFT + XB_REC])
        pair = torch.stack([g.xbuf[XB_DT:XB_DT + 2] for g in P]).amin(dim=0)
        for g in P:
            g.xbuf[XB_DT:XB_DT + 2].copy_(pair)

    def set_state(self, rho_global, mom_global, t_end=float("inf")):
        """rho/mom: the whole grid as 1-D device tensors."""
        import contextlib
        with torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext():
            self._set_state(rho_global, mom_global, t_end)

    def _set_state(self, rho_global, mom_global, t_end):
        for g in self.parts:
            r = torch.zeros(g.cap, dtype=torch.float64, device=rho_global.device)
            m = torch.zeros_like(r)
            r[:g.n] = rho_global[g.c0:g.c1]
            m[:g.n] = mom_global[g.c0:g.c1]
            g.ctx.set_state(r, m)
        self._exchange()
        for g in self.parts:
            g.ctx.step_finish(t_end, after_step=False)

    def _step_once(self, t_end):
        for g in self.parts:
            g.ctx.step_local(t_end)
        self._exchange()
        for g in self.parts:
            g.ctx.step_finish(t_end, after_step=True)

    def step(self, n_steps, t_end=float("inf"), graph_steps: int = 0):
        """graph_steps > 0: as RankGrid, the steps as replays of a captured CUDA graph (the
        contexts must have been created on a non-default torch stream, self.stream)."""
        import contextlib
        with torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext():
            if graph_steps and n_steps > 0:
                if self._graphs is None:
                    self._step_once(t_end)
                    n_steps -= 1
                    self._graphs = StepGraphs(self._step_once, self.stream, graph_steps)
                self._graphs.run(n_steps, t_end)
                return
            for _ in range(n_steps):
                self._step_once(t_end)

    def get_state(self):
        outs = [g.ctx.get_state() for g in self.parts]
        import numpy as np
        rho = np.concatenate([o["rho"][0, :int(o["n"][0])] for o in outs])
        mom = np.concatenate([o["mom"][0, :int(o["n"][0])] for o in outs])
        h = np.concatenate([o["h"][0, :int(o["n"][0])] for o in outs])
        return {"rho": rho, "mom": mom, "h": h, "t": [float(o["t"][0]) for o in outs],
                "status": [int(g.ctx.member_status()[0]) for g in self.parts]}
