"""DTS vs explicit LTS vs the Newton-like solve on the paper's cavitation (E2) and nucleation (E3)
tests, GPU and CPU oracle: local iterations and wall time (the paper's
P:1311-1332).  E3 with LTS needs ~1e6 sub-steps per large step: LTS runs E3 only to
the first arg (default 3e-5, 7 large steps), DTS and Newton run it to 3e-5 and to t_end = 5e-4.
Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2211_00705_b200 as P
from oracle import oracle as O
from conftest import eos_363K, read_golden
from paper_2211_00705_b200 import workloads as W

e3_t = float(sys.argv[1]) if len(sys.argv) > 1 else 3e-5


def setup(kind, mode):
    eos = eos_363K()
    g = read_golden("cavitation_363K.txt" if kind == "E2" else "nucleation_363K.txt")
    N, cap = 400, 416
    if kind == "E2":
        r = eos["rho0"] + (g["p_init"] - eos["p0"]) / eos["a_l"] ** 2; uL = -g["u_init"]
    else:
        r = g["p_init"] / eos["a_v2"]; uL = g["u_init"]
    prm = dict(W.PARAMS); prm["cfl"] = 0.5; prm["mode"] = mode
    rho = np.zeros((1, cap)); mom = np.zeros((1, cap))
    rho[0, :N] = r; mom[0, :N // 2] = r * uL; mom[0, N // 2:N] = -r * uL
    return eos, prm, N, cap, rho, mom


out = {}
for kind, t_end, modes in (("E2", 5e-4, (0, 2, 3)), ("E3", e3_t, (0, 2, 3)), ("E3full", 5e-4, (0, 3))):
    for mode, name in ((m, {0: "DTS", 2: "LTS", 3: "NEWTON"}[m]) for m in modes):
        eos, prm, N, cap, rho, mom = setup(kind[:2], mode)
        ctx = P.Context(eos, prm, 1, N, cap, -2.0, 2.0, stream=torch.cuda.current_stream())
        ctx.set_state(torch.tensor(rho, device="cuda"), torch.tensor(mom, device="cuda"))
        ctx.run_to(t_end)  # warm-up (module load, first launch)
        ctx.set_state(torch.tensor(rho, device="cuda"), torch.tensor(mom, device="cuda"))
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = ctx.run_to(t_end, stats=True)
        torch.cuda.synchronize(); tg = time.perf_counter() - t0
        s = O.Sim(eos, prm, 1, N, cap, -2.0, 2.0); s.set_state(rho, mom)
        t0 = time.perf_counter(); so = s.run_to(t_end); tc = time.perf_counter() - t0
        out[f"{kind}_{name}"] = {"t_end": t_end, "large_steps": st["steps"], "local_iterations_gpu": st["dts_iters"],
                                 "local_iterations_oracle": so["dts_iters"], "gpu_s": tg, "oracle_s": tc,
                                 "gpu_us_per_local_iteration": 1e6 * tg / max(st["dts_iters"], 1)}
        print(kind, name, out[f"{kind}_{name}"], flush=True)
for kind in ("E2", "E3"):
    d, l = out[f"{kind}_DTS"], out[f"{kind}_LTS"]
    out[f"{kind}_ratio"] = {"local_iterations_lts_over_dts": l["local_iterations_gpu"] / max(d["local_iterations_gpu"], 1),
                            "gpu_time_lts_over_dts": l["gpu_s"] / d["gpu_s"]}
for kind in ("E2", "E3", "E3full"):
    d, nt = out[f"{kind}_DTS"], out[f"{kind}_NEWTON"]
    out[f"{kind}_newton"] = {"evaluations_over_dts_iterations": nt["local_iterations_gpu"] / max(d["local_iterations_gpu"], 1),
                             "gpu_time_newton_over_dts": nt["gpu_s"] / d["gpu_s"]}
out["paper"] = {"E2": {"local_iterations": {"LTS": 1941, "DTS": 355}, "time_s": {"LTS": 4.93, "DTS": 2.94}, "cite": "P:1324-1325"},
                "E3": {"local_iterations": {"LTS": 27154016, "DTS": 1367460}, "time_s": {"LTS": 9811, "DTS": 509}, "cite": "P:1435-1436"}}
print(json.dumps(out))
