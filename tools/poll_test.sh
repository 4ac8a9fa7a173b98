cd $GRAFT_REPO_ROOT
cat > /tmp/pt.py <<'PY'
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2211_00705_b200 as P
from paper_2211_00705_b200 import workloads as W
w = W.c5(n_cells=30 * 940 + 311)
print("stream", torch.cuda.current_stream().cuda_stream, flush=True)
ctx = P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], w["x_left"], w["x_right"], stream=torch.cuda.current_stream(), layout=2)
ctx.set_state(torch.tensor(w["rho"], device="cuda"), torch.tensor(w["mom"], device="cuda"))
for k in range(3):
    t0 = time.time(); st = ctx.step(1, stats=True); print("step", k, time.time() - t0, st["creations"], flush=True)
PY
EIS_LIB=$PWD/build_variants/libeis_pd.so EIS_WIN_POLL_PER_SM=2 timeout 100 python /tmp/pt.py 2>&1 | sort | uniq -c | sort -rn | head -12
