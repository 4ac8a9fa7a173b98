"""Find the first step where GPU and oracle cell counts diverge for one C3 member (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
from oracle import oracle as O

mem = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
w = W.c3(members=np.array([mem]))
ctx = P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], 0.0, 1.0, stream=torch.cuda.current_stream())
ctx.set_state(torch.tensor(w["rho"], device="cuda"), torch.tensor(w["mom"], device="cuda"))
orc = O.Sim(w["eos"], w["params"], 1, w["N"], w["cap"], 0.0, 1.0)
orc.set_state(w["rho"], w["mom"])
h_av = 1.0 / w["N"]
for k in range(2000):
    g0 = ctx.get_state(); o0 = orc.get_state()
    ctx.step(1); orc.step(1)
    g = ctx.get_state(); o = orc.get_state()
    if g["n"][0] != o["n"][0]:
        n0 = int(o0["n"][0])
        print("first divergence at step", k + 1, "n gpu", g["n"][0], "orc", o["n"][0])
        # widths around thresholds before/after
        for name, s0, s1 in (("gpu", g0, g), ("orc", o0, o)):
            hs = s1["h"][0, :int(s1["n"][0])] / h_av
            idx = np.where((hs < 0.55) | (hs > 1.9))[0]
            print(name, "cells near thresholds after:", [(int(i), repr(hs[i])) for i in idx[:10]])
        # compare pre-step widths near interfaces
        d = np.abs(g0["h"][0, :n0] - o0["h"][0, :n0]) / h_av
        print("max pre-step width diff (h_av units)", d.max())
        for name, s0, s1 in (("gpu", g0, g), ("orc", o0, o)):
            print(name, "dt", repr(s1["t"][0] - s0["t"][0]), "post-step cells 744..752 h, h/h_av, rho:")
            for i in range(744, 753):
                print("  ", i, repr(s1["h"][0, i]), repr(s1["h"][0, i] / h_av), repr(s1["rho"][0, i]))
        break
else:
    print("no divergence in 2000 steps")
