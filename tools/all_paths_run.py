"""Small runs of every kernel family and mode (development smoke: resident, tiled ensembles and
grids, windows, DTS / LTS / Newton regions, interface reports, Lax batches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W


def run(w, layout=0, steps=None, t_end=None, mode=None, tile=0):
    if mode is not None:
        w["params"] = dict(w["params"]); w["params"]["mode"] = mode
    ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"],
                    stream=torch.cuda.current_stream(), layout=layout, tile_cells=tile)
    ctx.set_state(torch.tensor(w["rho"], device="cuda"), torch.tensor(w["mom"], device="cuda"))
    st = ctx.step(steps, stats=True) if steps else ctx.run_to(t_end, stats=True)
    ctx.get_state(); ctx.interfaces(); ctx.member_status()
    return st


print("C1", run(W.c1(), t_end=W.c1()["t_end"])["steps"])
print("C2 split", run(W.c2(), t_end=W.c2()["t_end"])["creations"])
print("C3 resident", run(W.c3(members=np.arange(4)), steps=60)["creations"])
print("C3 newton", run(W.c3(members=np.arange(4)), steps=60, mode=3)["dts_iters"])
print("C4 tiled", run(W.c4(members=np.arange(3)), steps=60, layout=2)["dts_iters"])
print("C4 tiled lts", run(W.c4(members=np.arange(3)), steps=30, layout=2, mode=2)["dts_iters"])
w = W.c5(n_cells=12 * 1400 + 311)
print("C5 tiled", run(w, steps=60, layout=2)["creations"])
print("C5 tiled newton", run(W.c5(n_cells=12 * 1400 + 311), steps=40, layout=2, mode=3)["regions"])
rho, mom, E, st = P.lax_run([dict(n=100, alpha=1e-2), dict(n=64, alpha=1.0, implicit_block=0, t_end=0.2)])
print("Lax", [s["status"] for s in st])
torch.cuda.synchronize()
print("done")
