"""C3 / C4 on the member-resident and the tiled layouts (dev tool): cell-updates/s."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
cfgs = sys.argv[1:] or ["c3:65536:500", "c4:16384:200"]
for spec in cfgs:
    cfg, M, K = spec.split(":"); M = int(M); K = int(K)
    w = W.c3(members=np.arange(M)) if cfg == "c3" else W.c4(members=np.arange(M))
    for layout in (1, 2):
        ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"],
                        stream=torch.cuda.current_stream(), layout=layout)
        r = torch.from_numpy(w["rho"]).cuda(); m = torch.from_numpy(w["mom"]).cuda()
        ctx.set_state(r, m); ctx.step(3); torch.cuda.synchronize(); ctx.set_state(r, m); torch.cuda.synchronize()
        t0 = time.time(); st = ctx.step(K, stats=True); dt = time.time() - t0
        bad = int((ctx.member_status() != 0).sum())
        print(f"{cfg} M={M} K={K} layout {layout}: {st['cell_updates'] / dt:.3e} cell-updates/s, {1e3 * dt / K:.3f} ms/step, "
              f"members not ok {bad}, creations {st['creations']}, dts {st['dts_iters']}", flush=True)
        del ctx
