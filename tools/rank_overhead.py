"""Host overhead of the rank-mode step loop (development tool): a small grid cut into 2 virtual
ranks on one GPU; wall time per step with GPU work ~ a few microseconds is the host cost of
step_local + exchange (device copies here, NCCL calls on a real box) + step_finish per rank."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
from paper_2211_00705_b200.decomp import VirtualRanks
n = 4 * 1400 * 2
w = W.c5(n_cells=n)
vr = VirtualRanks(w["eos"], w["params"], n, w["x_left"], w["x_right"], 2, tile=1400,
                  stream=torch.cuda.current_stream())
rho = torch.tensor(w["rho"][0, :n], device="cuda"); mom = torch.tensor(w["mom"][0, :n], device="cuda")
vr.set_state(rho, mom)
vr.step(20); torch.cuda.synchronize()
t0 = time.perf_counter(); vr.step(200); torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"virtual 2-rank step: {1e6 * dt / 200:.1f} us per step (both ranks, device-copy exchange)")
ctx = P.Context(w["eos"], w["params"], 1, n, w["cap"], w["x_left"], w["x_right"], stream=torch.cuda.current_stream(), layout=2)
ctx.set_state(torch.tensor(w["rho"], device="cuda"), torch.tensor(w["mom"], device="cuda"))
ctx.step(20); torch.cuda.synchronize()
t0 = time.perf_counter(); ctx.step(200); torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"one-rank eis_step(200): {1e6 * dt / 200:.1f} us per step")
t0 = time.perf_counter()
for _ in range(200): ctx.step(1)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"one-rank eis_step(1) x 200 from Python: {1e6 * dt / 200:.1f} us per step")
