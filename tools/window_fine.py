"""Finer phase breakdown of window full steps (development tool; a -DEIS_PHASE_CLOCK
-DEIS_FINE_CLOCK build via EIS_LIB, EIS_WINDOW_DEBUG).  usage: [WL=C4] python tools/window_fine.py step ..."""
import os, sys
os.environ["EIS_WINDOW_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
w = W.c4() if os.environ.get("WL") == "C4" else W.c5()
ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"],
                stream=torch.cuda.current_stream(), layout=2)
ctx.set_state(torch.from_numpy(w["rho"]).cuda(), torch.from_numpy(w["mom"]).cuda())
names = ["load+list", "S1", "P1", "A+dt", "S4..B", "S2 solves", "remesh+asm"]
done = 0
for target in [int(a) for a in (sys.argv[1:] or ["40", "450"])]:
    ctx.step(target - done); done = target
    ctx.step(1); done += 1
    d = ctx.window_diag().astype(np.float64)
    print(f"step {done}: windows {len(d)} total mean {d[:, 0].mean():.0f}")
    for i, nm in enumerate(names):
        v = d[:, 4 + i]
        print(f"   {nm:11s} mean {v.mean():8.0f}  p50 {np.percentile(v, 50):8.0f}  p90 {np.percentile(v, 90):8.0f}")
