"""Where the end-to-end time of the C5 bench goes (dev tool): set_state from pinned host
buffers, the K steps, get_state into pinned host buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200.decomp import RankGrid
from paper_2211_00705_b200 import workloads as W
K = int(sys.argv[1]) if len(sys.argv) > 1 else 500
w = W.c5()
rg = RankGrid(w["eos"], w["params"], w["N"], w["x_left"], w["x_right"], 0, 1, stream=torch.cuda.current_stream())
rho_h = torch.from_numpy(np.ascontiguousarray(w["rho"][0, :rg.cap])).pin_memory()
mom_h = torch.from_numpy(np.ascontiguousarray(w["mom"][0, :rg.cap])).pin_memory()
out = {k: torch.empty(rg.cap, dtype=torch.float64).pin_memory() for k in ("rho", "mom", "h")}
out["n"] = torch.empty(1, dtype=torch.int64).pin_memory(); out["t"] = torch.empty(1, dtype=torch.float64).pin_memory()
rg.set_state(rho_h, mom_h); rg.step(3); rg.ctx.get_state(out); torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); rg.set_state(rho_h, mom_h); torch.cuda.synchronize(); t1 = time.perf_counter()
    rg.step(K); torch.cuda.synchronize(); t2 = time.perf_counter()
    rg.ctx.get_state(out); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"set_state {t1 - t0:.3f} s  steps {t2 - t1:.3f} s  get_state {t3 - t2:.3f} s", flush=True)
