"""CPU-side checks of the boundary: libeis.so loads, exports every symbol include/eis.h
declares, and its host-side threshold routine (R3) agrees with the oracle's independent one.
No compute call needs a GPU here."""
import ctypes
import os
import re

import pytest

from conftest import ROOT, eos_363K


def _declared():
    src = open(os.path.join(ROOT, "include", "eis.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eis_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def P():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2211_00705_b200 as P
    return P


def test_header_and_binding_agree(P):
    assert sorted(P.SYMBOLS) == _declared()


def test_library_exports_every_declared_symbol(P):
    lib = ctypes.CDLL(P.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name


def test_sm100a_code_in_library(P):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("which", ["293K", "363K"])
def test_thresholds_match_oracle(P, oracle_mod, which):
    from paper_2211_00705_b200 import workloads as W
    eos = W.EOS_293K if which == "293K" else eos_363K()
    a = P.eis_thresholds_of(eos)
    b = oracle_mod.thresholds(eos)
    for k in ("rho_min", "rho_tilde", "p_tilde", "tau", "a_v"):
        assert a[k] == pytest.approx(b[k], rel=1e-12), k


def test_create_without_gpu_fails_loudly(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2211_00705_b200 import workloads as W
    w = W.c1()
    with pytest.raises(P.EisError):
        P.Context(w["eos"], w["params"], 1, w["N"], w["cap"], 0.0, 1.0)


def test_bad_arguments_rejected(P):
    from paper_2211_00705_b200 import workloads as W
    w = W.c1()
    with pytest.raises(P.EisError):
        P.Context(w["eos"], w["params"], 1, w["N"], w["N"] - 1, 0.0, 1.0)  # capacity < N
    bad = dict(w["params"])
    bad["cfl"] = -1.0
    with pytest.raises(P.EisError):
        P.Context(w["eos"], bad, 1, w["N"], w["cap"], 0.0, 1.0)
