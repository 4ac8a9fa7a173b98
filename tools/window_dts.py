"""DTS cost breakdown of window full steps (development tool; a -DEIS_DTS_CLOCK build via
EIS_LIB, EIS_WINDOW_DEBUG): cycles in boundary-solve rounds and in updates per DTS iteration,
Newton iterations per solve.  usage: [WL=C4] python tools/window_dts.py step ..."""
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
done = 0
for target in [int(a) for a in (sys.argv[1:] or ["1", "50", "1000"])]:
    ctx.step(target - done); done = target
    ctx.step(1); done += 1
    d = ctx.window_diag().astype(np.float64)
    tot, it = d[:, 0], d[:, 1]
    solve, upd, its, blk, nit, nsol = d[:, 5], d[:, 6], d[:, 7], d[:, 8], d[:, 9], d[:, 10]
    m = its > 0
    print(f"step {done}: windows {len(d)} with DTS {m.sum()} | window cycles mean {tot.mean():.0f} | "
          f"DTS its/window {its[m].mean():.1f} blocks {blk[m].mean():.2f} | per iteration: solve rounds "
          f"{(solve[m] / its[m]).mean():.0f} update {(upd[m] / its[m]).mean():.0f} cycles | DTS share "
          f"{((solve + upd)[m] / tot[m]).mean():.2f} | Newton its per solve {nit.sum() / max(nsol.sum(), 1):.2f}", flush=True)
