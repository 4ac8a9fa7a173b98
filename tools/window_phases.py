"""Phase breakdown of window full steps (development tool; needs a -DEIS_PHASE_CLOCK build via
EIS_LIB and EIS_WINDOW_DEBUG).  Reads the extra clocks behind the window diagnostics."""
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
nt = ctx.tile_info()["n_tiles"]
done = 0
for target in [int(a) for a in (sys.argv[1:] or ["1", "40", "200"])]:
    ctx.step(target - done); done = target
    ctx.step(1); done += 1
    d = ctx.window_diag()
    n = len(d)
    ph = d[:, 5:11]
    names = ["load+list", "start->A", "A->B", "S4 (DTS)", "B->end", "assembly"]
    print(f"step {done}: windows {n}, total p50 {np.percentile(d[:, 0], 50):.0f}, dts mean {d[:, 1].mean():.1f}")
    for i, nm in enumerate(names):
        print(f"   {nm:14s} mean {ph[:, i].mean():9.0f}  p50 {np.percentile(ph[:, i], 50):9.0f}  p90 {np.percentile(ph[:, i], 90):9.0f}")
