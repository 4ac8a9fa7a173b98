"""DTS decision parity probe (dev tool): per member, GPU vs oracle DTS iteration totals, boundary
solve counts, regions, relative L1 and element-wise errors, for several Newton-gate settings.

  python tools/dts_probe.py [settings...]   settings: name=STOL:LIN_GTOL (env knobs of eis_create)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import paper_2211_00705_b200 as P
from oracle import oracle as O
from paper_2211_00705_b200 import workloads as W
from conftest import eos_363K, read_golden


def e_workload(kind):
    eos = eos_363K()
    g_ = read_golden("cavitation_363K.txt" if kind == "E2" else "nucleation_363K.txt")
    N, cap = 400, 416
    prm = dict(W.PARAMS); prm["cfl"] = 0.5
    rho = np.zeros((1, cap)); mom = np.zeros((1, cap))
    if kind == "E2":
        r = eos["rho0"] + (g_["p_init"] - eos["p0"]) / eos["a_l"] ** 2
        rho[0, :N] = r; mom[0, :N // 2] = -r * g_["u_init"]; mom[0, N // 2:N] = r * g_["u_init"]
    else:
        r = g_["p_init"] / eos["a_v2"]
        rho[0, :N] = r; mom[0, :N // 2] = r * g_["u_init"]; mom[0, N // 2:N] = -r * g_["u_init"]
    return dict(eos=eos, params=prm, M=1, N=N, cap=cap, x_left=-2.0, x_right=2.0, rho=rho, mom=mom, t_end=5e-4)


CASES = {
    "E2": (lambda: e_workload("E2"), None, 0, 0),
    "E3": (lambda: e_workload("E3"), None, 0, 0),
    "C2": (lambda: W.c2(), None, 0, 0),
    "C3": (lambda: W.c3(members=np.array([0, 1, 2, 3, 17, 100, 4097, 30000, 65535])), 300, 0, 0),
    "C4": (lambda: W.c4(members=np.arange(16)), 300, 0, 0),
    "C5": (lambda: W.c5(n_cells=1 << 16), 200, 2, 1024),
}


def run_gpu(w, steps, layout, tile):
    ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"],
                    stream=torch.cuda.current_stream(), layout=layout, tile_cells=tile)
    ctx.set_state(torch.tensor(w["rho"], device="cuda"), torch.tensor(w["mom"], device="cuda"))
    st = ctx.step(steps, stats=True) if steps else ctx.run_to(w["t_end"], stats=True)
    g = ctx.get_state()
    g["mstats"] = ctx.member_stats()
    g["status"] = ctx.member_status()
    return g


def run_orc(w, steps):
    s = O.Sim(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"])
    s.set_state(w["rho"], w["mom"])
    st = s.step(steps) if steps else s.run_to(w["t_end"])
    o = s.get_state()
    o["mstats"] = [s.member_stats(m) for m in range(w["M"])]
    return o


def compare(g, o, M):
    rows = []
    for m in range(M):
        n = int(o["n"][m]); ng = int(g["n"][m])
        r = {"m": m, "n_equal": n == ng}
        gs, os_ = g["mstats"][m], o["mstats"][m]
        for k in ("dts_iters", "iface_solves", "regions", "creations", "merges", "splits", "decision_margin_warnings"):
            r[k] = [int(gs[k]), int(os_[k])]
        if n == ng:
            for k in ("rho", "mom"):
                a, b = g[k][m, :n], o[k][m, :n]
                r["l1_" + k] = float(np.sum(o["h"][m, :n] * np.abs(a - b)) / np.sum(o["h"][m, :n] * np.abs(b)))
                r["el_" + k] = float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))
            r["el_h"] = float(np.max(np.abs(g["h"][m, :n] - o["h"][m, :n]) / o["h"][m, :n]))
        rows.append(r)
    return rows


def main():
    settings = sys.argv[1:] or ["base=:", "stol8=1e-8:", "stol8_nolin=1e-8:0"]
    cases = os.environ.get("CASES", ",".join(CASES)).split(",")
    out = {}
    for cname in cases:
        mk, steps, layout, tile = CASES[cname]
        w = mk()
        t0 = time.time()
        o = run_orc(w, steps)
        to = time.time() - t0
        for s in settings:
            name, kv = s.split("=")
            stol, lg = kv.split(":")
            for k, v in (("EIS_NEWTON_STOL", stol), ("EIS_LIN_GTOL", lg)):
                if v:
                    os.environ[k] = v
                else:
                    os.environ.pop(k, None)
            t0 = time.time()
            g = run_gpu(w, steps, layout, tile)
            torch.cuda.synchronize()
            tg = time.time() - t0
            rows = compare(g, o, w["M"])
            mism = sum(r["dts_iters"][0] != r["dts_iters"][1] for r in rows)
            smism = sum(r["iface_solves"][0] != r["iface_solves"][1] for r in rows)
            rec = {"case": cname, "setting": name, "oracle_s": round(to, 2), "gpu_s": round(tg, 2),
                   "dts_mismatch_members": mism, "solve_mismatch_members": smism, "members": w["M"],
                   "dts_total": [sum(r["dts_iters"][0] for r in rows), sum(r["dts_iters"][1] for r in rows)],
                   "max_el_rho": max(r.get("el_rho", -1) for r in rows), "max_el_mom": max(r.get("el_mom", -1) for r in rows),
                   "max_l1_rho": max(r.get("l1_rho", -1) for r in rows), "max_l1_mom": max(r.get("l1_mom", -1) for r in rows),
                   "status_bad": int((g["status"] != 0).sum()), "rows": rows,
                   "margins": [sum(r["decision_margin_warnings"][0] for r in rows), sum(r["decision_margin_warnings"][1] for r in rows)],
                   "mismatch_unflagged": sum(r["dts_iters"][0] != r["dts_iters"][1] and r["decision_margin_warnings"] == [0, 0] for r in rows)}
            print(json.dumps({k: v for k, v in rec.items() if k != "rows"}), flush=True)
            out[f"{cname}/{name}"] = rec
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "dts_probe.json"), "w"), indent=1)


if __name__ == "__main__" and not os.environ.get("ONESTEP"):
    main()


def onestep(cname, steps_override=None):
    """Per step: the GPU starts from the oracle's state, both take one large step; per member the
    DTS counts must agree unless either side logged a decision-margin warning in that step."""
    mk, steps, layout, tile = CASES[cname]
    w = mk()
    K = steps_override or steps or 150
    s = O.Sim(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"])
    s.set_state(w["rho"], w["mom"])
    ctx = P.Context(w["eos"], w["params"], w["M"], w["N"], w["cap"], w["x_left"], w["x_right"],
                    stream=torch.cuda.current_stream(), layout=layout, tile_cells=tile)
    M = w["M"]
    keys = ("dts_iters", "iface_solves", "regions", "creations", "decision_margin_warnings")
    prev = [dict((k, 0) for k in keys) for _ in range(M)]
    tot = {"member_steps": 0, "dts_mismatch": 0, "justified": 0, "unjustified": 0, "solve_mismatch": 0,
           "margin_orc": 0, "margin_gpu": 0, "max_el": 0.0, "max_el_nonblock": 0.0, "unjust_list": []}
    for step in range(K):
        o = s.get_state()
        ctx.set_state(o["rho"], o["mom"], width=o["h"], n_cells=o["n"].astype(np.int64))
        ctx.step(1)
        s.step(1)
        gms = ctx.member_stats()
        oms = [s.member_stats(m) for m in range(M)]
        g = ctx.get_state(); o2 = s.get_state()
        for m in range(M):
            d_o = {k: oms[m][k] - prev[m][k] for k in keys}
            d_g = {k: gms[m][k] for k in keys}  # set_state resets the GPU counters
            prev[m] = {k: oms[m][k] for k in keys}
            tot["member_steps"] += 1
            tot["margin_orc"] += d_o["decision_margin_warnings"]; tot["margin_gpu"] += d_g["decision_margin_warnings"]
            if d_g["iface_solves"] != d_o["iface_solves"]:
                tot["solve_mismatch"] += 1
            if d_g["dts_iters"] != d_o["dts_iters"]:
                tot["dts_mismatch"] += 1
                if d_o["decision_margin_warnings"] + d_g["decision_margin_warnings"] > 0:
                    tot["justified"] += 1
                else:
                    tot["unjustified"] += 1
                    if len(tot["unjust_list"]) < 20:
                        tot["unjust_list"].append([step, m, d_g["dts_iters"], d_o["dts_iters"]])
            n = int(o2["n"][m])
            if int(g["n"][m]) == n:
                for k in ("rho", "mom"):
                    e = np.abs(g[k][m, :n] - o2[k][m, :n]) / np.maximum(np.abs(o2[k][m, :n]), 1.0)
                    tot["max_el"] = max(tot["max_el"], float(e.max()))
                    wide = o2["h"][m, :n] >= 0.5 * (w["x_right"] - w["x_left"]) / w["N"]
                    if wide.any():
                        tot["max_el_nonblock"] = max(tot["max_el_nonblock"], float(e[wide].max()))
    tot["case"] = cname
    print(json.dumps(tot), flush=True)
    return tot


if __name__ == "__main__" and os.environ.get("ONESTEP"):
    for c in os.environ["ONESTEP"].split(","):
        onestep(c)
