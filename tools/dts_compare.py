"""Per-step DTS iteration counts, GPU vs oracle, on the paper's nucleation test (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from oracle import oracle as O
from conftest import eos_363K, read_golden
from paper_2211_00705_b200 import workloads as W
eos = eos_363K()
g_ = read_golden("nucleation_363K.txt")
N, cap = 400, 416
r = g_["p_init"] / eos["a_v2"]
prm = dict(W.PARAMS); prm["cfl"] = 0.5
rho = np.zeros((1, cap)); mom = np.zeros((1, cap))
rho[0, :N] = r; mom[0, :N // 2] = r * g_["u_init"]; mom[0, N // 2:N] = -r * g_["u_init"]
ctx = P.Context(eos, prm, 1, N, cap, -2.0, 2.0, stream=torch.cuda.current_stream())
ctx.set_state(torch.tensor(rho, device="cuda"), torch.tensor(mom, device="cuda"))
s = O.Sim(eos, prm, 1, N, cap, -2.0, 2.0)
s.set_state(rho, mom)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
pg = po = pr = qr = 0
for k in range(K):
    a = ctx.step(1, stats=True); b = s.step(1)
    gs, os_ = ctx.get_state(), s.get_state()
    n = int(gs["n"][0])
    drho = np.max(np.abs(gs["rho"][0, :n] - os_["rho"][0, :n]) / np.maximum(np.abs(os_["rho"][0, :n]), 1e-300))
    i = int(np.argmin(np.abs(np.arange(n) - n // 2) + 1e9 * (gs["h"][0, :n] > 0.5 * 1e-2)))
    print(f"step {k+1}: gpu dts {a['dts_iters'] - pg:7d} reg {a['regions'] - pr:3d} | oracle {b['dts_iters'] - po:7d} reg {b['regions'] - qr:3d} | max rel drho {drho:.2e} | n {n} {int(os_['n'][0])} | narrow cells gpu {np.nonzero(gs['h'][0, :n] < 5e-3)[0].tolist()} h {gs['h'][0, gs['h'][0, :n].argmin()]:.3e} oracle {np.nonzero(os_['h'][0, :n] < 5e-3)[0].tolist()} h {os_['h'][0, os_['h'][0, :n].argmin()]:.3e}", flush=True)
    pg, po, pr, qr = a["dts_iters"], b["dts_iters"], a["regions"], b["regions"]
