"""Full-size C5 on one GPU: 2^27 cells, K steps, device-side timing (development tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 960
t0 = time.time()
w = W.c5()
print("generated", time.time() - t0, flush=True)
ctx = P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], w["x_left"], w["x_right"],
                stream=torch.cuda.current_stream(), layout=2, tile_cells=tile)
rho = torch.from_numpy(w["rho"]).cuda(); mom = torch.from_numpy(w["mom"]).cuda()
ctx.set_state(rho, mom)
ctx.step(3)
torch.cuda.synchronize()
ctx.set_state(rho, mom)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.step(K)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
st = ctx.step(0, stats=True)
print(f"K={K} ms/step={ms / K:.3f} cell-updates/s={st['cell_updates'] / (ms * 1e-3):.3e} status={ctx.member_status()} stats={st}")
print("GB/s at 48 B/cell:", 48 * st["cell_updates"] / (ms * 1e-3) / 1e9)
