"""C5-like grid: tiled GPU layout vs the oracle (and vs the resident layout when it fits)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
tile = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
w = W.c5(n_cells=n)


def gpu(layout):
    ctx = P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], w["x_left"], w["x_right"],
                    stream=torch.cuda.current_stream(), layout=layout, tile_cells=tile if layout == 2 else 0)
    ctx.set_state(torch.tensor(w["rho"], device="cuda"), torch.tensor(w["mom"], device="cuda"))
    torch.cuda.synchronize(); t0 = time.time()
    st = ctx.step(steps, stats=True)
    tg = time.time() - t0
    g = ctx.get_state()
    g["status"] = ctx.member_status(); g["ifc"] = ctx.interfaces(); g["st"] = st
    return g, tg


orc = O.Sim(w["eos"], w["params"], 1, w["N"], w["cap"], w["x_left"], w["x_right"])
orc.set_state(w["rho"], w["mom"])
t0 = time.time(); so = orc.step(steps); to = time.time() - t0
o = orc.get_state(); o["status"] = orc.member_status(); o["ifc"] = orc.interfaces()
print("oracle", so, f"{to:.2f}s", "status", o["status"])
layouts = [2] + ([1] if w["cap"] <= 16384 else [])
for lay in layouts:
    g, tg = gpu(lay)
    nn = int(o["n"][0])
    msg = f"layout {lay}: status {g['status']} n gpu {g['n'][0]} orc {nn} time {tg:.3f}s stats {g['st']}"
    if g["n"][0] == nn:
        for k in ("rho", "mom"):
            den = np.sum(o["h"][0, :nn] * np.abs(o[k][0, :nn]))
            err = np.sum(o["h"][0, :nn] * np.abs(g[k][0, :nn] - o[k][0, :nn])) / den
            msg += f" relL1[{k}]={err:.3e}"
        msg += f" ifc {len(g['ifc'])}/{len(o['ifc'])}"
        if len(g["ifc"]) == len(o["ifc"]):
            msg += f" max|dx|={max([abs(a['x'] - b['x']) for a, b in zip(g['ifc'], o['ifc'])], default=0):.3e}"
    print(msg)
