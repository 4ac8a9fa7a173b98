"""Dev diagnostics: the K=5 block case and the full-size C5 prefix comparison, cell by cell."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
from oracle import oracle as O
import test_gpu_parity as T

what = sys.argv[1]
if what == "k5":
    w = T._two_bubbles(M=2)
    for steps in (1, 2, 5, 30):
        ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"], stream=torch.cuda.current_stream(), layout=1)
        ctx.set_state(w["rho"], w["mom"], width=w["h"]); ctx.step(steps)
        g = ctx.get_state(); gm = ctx.member_stats()
        s = O.Sim(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"]); s.set_state(w["rho"], w["mom"], width=w["h"]); s.step(steps)
        o = s.get_state()
        for m in range(2):
            n = int(o["n"][m])
            print("steps", steps, "m", m, "n", n, int(g["n"][m]), "dts g/o", gm[m]["dts_iters"], s.member_stats(m)["dts_iters"],
                  "solves", gm[m]["iface_solves"], s.member_stats(m)["iface_solves"], "marg", gm[m]["decision_margin_warnings"], s.member_stats(m)["decision_margin_warnings"])
            for i in range(97, 106):
                print("   ", i, "h %.6e %.6e" % (g["h"][m, i], o["h"][m, i]), "rho %.15e %.15e" % (g["rho"][m, i], o["rho"][m, i]), "mom %.15e %.15e" % (g["mom"][m, i], o["mom"][m, i]))
elif what == "c5pre":
    S, steps = 1 << 20, int(sys.argv[2]) if len(sys.argv) > 2 else 20
    w = W.c5()
    ctx = P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], w["x_left"], w["x_right"], stream=torch.cuda.current_stream(), layout=2, tile_cells=1400)
    ctx.set_state(torch.from_numpy(w["rho"]).cuda(), torch.from_numpy(w["mom"]).cuda())
    ctx.step(steps)
    g = ctx.get_state()
    del w
    wp = W.c5(n_cells=S)
    s = O.Sim(wp["eos"], wp["params"], 1, wp["N"], wp["cap"], wp["x_left"], wp["x_right"]); s.set_state(wp["rho"], wp["mom"]); s.step(steps)
    o = s.get_state()
    cut = S - 600
    for k in ("rho", "mom", "h"):
        e = np.abs(g[k][0, :cut] - o[k][0, :cut]) / np.maximum(np.abs(o[k][0, :cut]), 1.0)
        bad = np.nonzero(e > 1e-10)[0]
        print(k, "max", e.max(), "n bad", len(bad), "first", bad[:10])
        if len(bad):
            i = bad[0]
            for j in range(max(0, i - 3), i + 4):
                print("   ", j, "g", g["rho"][0, j], g["h"][0, j], "o", o["rho"][0, j], o["h"][0, j])
