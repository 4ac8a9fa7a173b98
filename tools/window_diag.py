"""Distribution of window full-step latencies on C5 / C4 (development tool): EIS_WINDOW_DEBUG.
usage: [WL=C4] python tools/window_diag.py step ..."""
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
for target in [int(a) for a in (sys.argv[1:] or ["1", "2", "5", "40", "200", "500"])]:
    ctx.step(target - done); done = target
    ctx.set_timing(True); ctx.step(1); done += 1
    kt = ctx.get_timing(); ctx.set_timing(False)
    d = ctx.window_diag()
    cyc, it, wc, nb, t0 = d[:, :5].T
    span = (t0 + cyc).max() - t0.min()
    q = np.percentile(cyc, [50, 90, 99, 100])
    print(f"step {done}: windows {len(d)} fast {kt['fast_ms']:.3f} ms win {kt['window_ms']:.3f} ms slow {kt['tile_ms']:.3f} ms | "
          f"cycles p50/p90/p99/max {q.astype(int)} sum {cyc.sum():.3e} span {span:.3e} | dts it mean {it.mean():.1f} max {it.max()} | "
          f"cells mean {wc.mean():.0f} max {wc.max()} | bnd mean {nb.mean():.1f}", flush=True)
    big = np.argsort(-cyc)[:3]
    print("   slowest:", [(int(cyc[i]), int(it[i]), int(wc[i]), int(nb[i])) for i in big])
