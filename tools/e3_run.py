"""The paper's nucleation test (E3) on the GPU for a given end time (dev tool: DTS latency)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from conftest import eos_363K, read_golden
from paper_2211_00705_b200 import workloads as W
t_end = float(sys.argv[1]) if len(sys.argv) > 1 else 5e-5
eos = eos_363K(); g_ = read_golden("nucleation_363K.txt")
N, cap = 400, 416
r = g_["p_init"] / eos["a_v2"]
prm = dict(W.PARAMS); prm["cfl"] = 0.5
rho = np.zeros((1, cap)); mom = np.zeros((1, cap))
rho[0, :N] = r; mom[0, :N // 2] = r * g_["u_init"]; mom[0, N // 2:N] = -r * g_["u_init"]
ctx = P.Context(eos, prm, 1, N, cap, -2.0, 2.0, stream=torch.cuda.current_stream())
ctx.set_state(torch.tensor(rho, device="cuda"), torch.tensor(mom, device="cuda"))
torch.cuda.synchronize(); t0 = time.time()
st = ctx.run_to(t_end, stats=True)
torch.cuda.synchronize(); dt = time.time() - t0
print(f"E3 to {t_end}: {st['steps']} steps, {st['dts_iters']} DTS iterations, {dt:.3f} s, {1e6 * dt / max(st['dts_iters'], 1):.2f} us/iteration")
