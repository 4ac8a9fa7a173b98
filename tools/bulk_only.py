"""Throughput of the resident kernel on single-phase members (no boundaries, no creation):
the bulk passes alone (development tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W

M = int(os.environ.get("BULK_M", "65536")); N, K = 1024, int(sys.argv[1]) if len(sys.argv) > 1 else 500
w = W.c3(M=M)
u = np.where(np.arange(N) < N // 2, -2.0, 2.0)  # gentle expansion: no cavitation
w["mom"][:, :N] = w["rho"][:, :N] * u[None, :]
ctx = P.Context(w["eos"], w["params"], M, N, w["cap"], 0.0, 1.0, stream=torch.cuda.current_stream(), threads=int(os.environ.get("THREADS", "0")))
rho = torch.from_numpy(w["rho"]).cuda(); mom = torch.from_numpy(w["mom"]).cuda()
ctx.set_state(rho, mom); ctx.step(3); torch.cuda.synchronize(); ctx.set_state(rho, mom)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ctx.step(K); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
st = ctx.step(0, stats=True)
print(f"bulk-only: {st['cell_updates'] / (ms * 1e-3):.3e} cell-updates/s, {ms / K:.3f} ms/step, creations {st['creations']}")
