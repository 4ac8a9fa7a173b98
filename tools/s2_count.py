"""Newton iterations of the explicit boundary solves (S2) in C5 window steps at steady state
(development tool; a -DEIS_DTS_CLOCK -DEIS_S2_COUNT build via EIS_LIB).  Measured after R14d:
1.0 iteration (one evaluation) per warm-started solve."""
import os, sys
os.environ["EIS_WINDOW_DEBUG"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
w = W.c5()
ctx = P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], w["x_left"], w["x_right"], stream=torch.cuda.current_stream(), layout=2)
ctx.set_state(torch.from_numpy(w["rho"]).cuda(), torch.from_numpy(w["mom"]).cuda())
ctx.step(450); ctx.step(1)
d = ctx.window_diag().astype(np.float64)
warm, nsol, nit = d[:, 7].sum(), d[:, 8].sum(), d[:, 9].sum()
print("windows", len(d), "S2 solves", nsol, "warm", warm, "Newton its per S2 solve", nit / max(nsol, 1))
