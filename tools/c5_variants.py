"""C5 variants on one GPU (development tool): recipe | uniform (rho=1000, u=0: the pure bulk
floor of the tiled step) | calm (segments with |v| <= 5 m/s: no creation).  Device-timed."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W

var = sys.argv[1] if len(sys.argv) > 1 else "recipe"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 27
tile = int(os.environ.get("TILE", "940"))
w = W.c5(n_cells=n)
if var == "uniform":
    w["rho"][0, :n] = 1000.0
    w["mom"][0, :n] = 0.0
elif var == "calm":
    w["mom"][0, :n] = w["mom"][0, :n] * (5.0 / 150.0)
ctx = P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], w["x_left"], w["x_right"],
                stream=torch.cuda.current_stream(), layout=2, tile_cells=tile)
rho = torch.from_numpy(w["rho"]).cuda(); mom = torch.from_numpy(w["mom"]).cuda()
ctx.set_state(rho, mom)
ctx.step(3)
torch.cuda.synchronize()
ctx.set_state(rho, mom)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if os.environ.get("PERSTEP"):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    ev[0].record()
    for i in range(K):
        ctx.step(1)
        ev[i + 1].record()
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
    ms = sum(per)
    print("per-step ms:", " ".join(f"{x:.2f}" for x in per))
else:
    e0.record()
    ctx.step(K)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
st = ctx.step(0, stats=True)
print(ctx.tile_info()); print(f"{var} n={n} tile={tile} K={K} ms/step={ms / K:.3f} cu/s={st['cell_updates'] / (ms * 1e-3):.3e} "
      f"GB/s@48B={48 * st['cell_updates'] / (ms * 1e-3) / 1e9:.0f} status={ctx.member_status()} stats={st}", flush=True)
