"""Quick GPU-vs-oracle probe (development tool): prints per-config parity numbers."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
from oracle import oracle as O


def run(w, steps=None, t_end=None, threads=0):
    ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"],
                    stream=torch.cuda.current_stream(), threads=threads)
    ctx.set_state(torch.tensor(w["rho"], device="cuda"), torch.tensor(w["mom"], device="cuda"))
    t0 = time.time()
    st = ctx.step(steps, stats=True) if steps else ctx.run_to(t_end, stats=True)
    tg = time.time() - t0
    g = ctx.get_state()
    g["status"] = ctx.member_status()
    g["ifc"] = ctx.interfaces()
    orc = O.Sim(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"])
    orc.set_state(w["rho"], w["mom"])
    t0 = time.time()
    so = orc.step(steps) if steps else orc.run_to(t_end)
    to = time.time() - t0
    o = orc.get_state()
    o["status"] = orc.member_status()
    o["ifc"] = orc.interfaces()
    return g, o, st, so, tg, to


def report(name, g, o, st, so, tg, to):
    M = len(g["n"])
    worst = 0.0
    bad = []
    for m in range(M):
        if g["n"][m] != o["n"][m] or g["status"][m] != o["status"][m]:
            bad.append((m, int(g["n"][m]), int(o["n"][m]), int(g["status"][m]), int(o["status"][m])))
            continue
        n = int(o["n"][m])
        for k in ("rho", "mom"):
            den = np.sum(o["h"][m, :n] * np.abs(o[k][m, :n]))
            err = np.sum(o["h"][m, :n] * np.abs(g[k][m, :n] - o[k][m, :n])) / den
            worst = max(worst, err)
    print(f"{name}: M={M} worst relL1={worst:.3e} mismatched(n/status)={bad[:5]} ({len(bad)})")
    print(f"   gpu stats {st}  {tg:.3f}s")
    print(f"   orc stats {so}  {to:.3f}s")
    xi = [(a['x'], b['x']) for a, b in zip(g['ifc'], o['ifc'])]
    print(f"   interfaces gpu={len(g['ifc'])} orc={len(o['ifc'])} max|dx|={max([abs(a-b) for a,b in xi], default=0):.3e}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c2e", "c3", "c4"]
    if "c1" in which:
        w = W.c1(); report("C1", *run(w, t_end=w["t_end"]))
    if "c2" in which:
        w = W.c2(); report("C2 split", *run(w, t_end=w["t_end"]))
    if "c2e" in which:
        w = W.c2(W.MODE_EXPLICIT); report("C2 explicit", *run(w, t_end=w["t_end"]))
    if "c3" in which:
        w = W.c3(members=np.arange(32)); report("C3[0:32] 300 steps", *run(w, steps=300))
    if "c4" in which:
        w = W.c4(members=np.arange(16)); report("C4[0:16] 100 steps", *run(w, steps=100))
