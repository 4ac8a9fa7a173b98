"""GPU parity of the Lax shock-tube batches (eis_lax_run, paper_2211_00705_b200/csrc/eis_lax.cuh:
its own exact Riemann solver and the hot path's DTS warp loop, eis_dts.cuh)
against the CPU oracle (oracle/lax.c): final conserved states within relative L1 1e-9 per
component, identical step counts and DTS iteration counts (unless a stop decision was marginal), on the cases of
tab:iterations (tests/golden/lax_iterations.txt) run as one batch, explicit-only cases and seeded
Riemann data."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REL_L1 = 1e-9


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2211_00705_b200 as P
    return P


def _cases():
    cs = []
    for th in (0.9, 0.1):
        for N in (100, 200, 400):
            for a in (1e-2, 1e-4, 1e-6):
                cs.append(dict(n=N, alpha=a, theta_nb=th))
    for N in (100, 200, 400):
        cs.append(dict(n=N, alpha=1e-2, theta_nb=1e-2))
    cs.append(dict(n=100, alpha=1.0, implicit_block=0))
    cs.append(dict(n=400, alpha=1.0, implicit_block=0))
    cs.append(dict(n=64, alpha=0.5, implicit_block=0, t_end=0.5))
    rng = np.random.default_rng(2211)
    for i in range(6):  # seeded Riemann data, ragged N
        cs.append(dict(n=int(rng.integers(3, 160)) * 2, alpha=float(10 ** rng.uniform(-6, -1)),
                       theta_nb=float(rng.uniform(0.05, 1.0)), rho_l=float(rng.uniform(0.2, 2)),
                       u_l=float(rng.uniform(-1, 1)), p_l=float(rng.uniform(0.2, 4)), rho_r=float(rng.uniform(0.2, 2)),
                       u_r=float(rng.uniform(-1, 1)), p_r=float(rng.uniform(0.2, 4)), t_end=float(rng.uniform(0.2, 1))))
    return cs


def _rel_l1(a, b):
    return np.abs(a - b).sum() / max(np.abs(b).sum(), 1e-300)


def _oracle(O, kw):
    d = {k: v for k, v in kw.items() if k != "dts_loop"}
    return O.lax_run(O.lax_case(**d))


@pytest.mark.parametrize("loop", [0, 1])
def test_lax_batch_parity(P, oracle_mod, loop):
    """loop 0: Algorithm 2 by the warp loop (dts_warp), 1: by the one-thread loop (dts_thread)."""
    O = oracle_mod
    cases = [dict(c, dts_loop=loop) for c in _cases()]
    rho, mom, E, stats = P.lax_run(cases)
    rho, mom, E = rho.cpu().numpy(), mom.cpu().numpy(), E.cpu().numpy()
    for i, kw in enumerate(cases):
        r, m, e, xf, so = _oracle(O, kw)
        sg = stats[i]
        assert sg["status"] == 0 and so["status"] == 0, (kw, sg, so)
        assert sg["steps"] == so["steps"], (kw, sg, so)
        # the same DTS stop decisions, except where a decision sat within its rounding-error
        # bound (the GPU's own margin count; the two Riemann solvers differ in roundoff)
        if sg["margins"] == 0:
            assert sg["dts_iters"] == so["dts_iters"] and sg["dts_max"] == so["dts_max"], (kw, sg, so)
            assert sg["riemann_solves"] == so["riemann_solves"], (kw, sg, so)
        else:
            assert abs(sg["dts_iters"] - so["dts_iters"]) <= sg["margins"], (kw, sg, so)
        assert sg["t"] == pytest.approx(so["t"], rel=1e-13)
        nc = kw["n"] + 1
        for got, ref in ((rho[i, :nc], r), (mom[i, :nc], m), (E[i, :nc], e)):
            assert _rel_l1(got, ref) <= REL_L1, (kw, _rel_l1(got, ref))


def test_lax_theta_alpha_at_scale(P, oracle_mod):
    """theta_{k+-1} = alpha = 1e-4 (~4e4 DTS iterations per step): GPU vs oracle at
    N = 100, and the printed O(1/alpha) growth for N = 100, 200, 400 within the R23 factor 1.5."""
    O = oracle_mod
    cases = [dict(n=N, alpha=1e-4, theta_nb=1e-4) for N in (100, 200, 400)]
    rho, mom, E, stats = P.lax_run(cases)
    printed = {100: 43470, 200: 34356, 400: 24178}  # tests/golden/lax_iterations.txt
    for kw, sg in zip(cases, stats):
        assert sg["status"] == 0
        avg = sg["dts_iters"] / sg["steps"]
        assert printed[kw["n"]] / 1.5 <= avg <= printed[kw["n"]] * 1.5, (kw, avg)
    r, m, e, xf, so = _oracle(O, cases[0])
    assert stats[0]["steps"] == so["steps"]
    assert abs(stats[0]["dts_iters"] - so["dts_iters"]) <= stats[0]["margins"], (stats[0], so)
    assert _rel_l1(rho[0, :101].cpu().numpy(), r) <= REL_L1


def test_lax_bad_arguments(P):
    for bad in (dict(n=101), dict(n=4), dict(alpha=0.0), dict(theta_nb=-1.0), dict(n=5000)):
        with pytest.raises(P.EisError):
            P.lax_run([bad])


def test_lax_maximum_mesh_and_many_cases(P, oracle_mod):
    """The largest mesh a case may use (N = 4094, 4095 cells in shared memory) next to 200 small
    seeded cases in one launch; the big case and a sample of the small ones against the oracle."""
    O = oracle_mod
    rng = np.random.default_rng(7)
    cases = [dict(n=4094, alpha=1e-3, theta_nb=0.9, t_end=0.05)]
    for i in range(200):
        cases.append(dict(n=int(rng.integers(3, 60)) * 2, alpha=float(10 ** rng.uniform(-5, -1)),
                          theta_nb=float(rng.uniform(0.1, 1.0)), t_end=float(rng.uniform(0.05, 0.5))))
    rho, mom, E, stats = P.lax_run(cases)
    assert all(s["status"] == 0 for s in stats)
    for i in [0] + list(range(1, 201, 20)):
        kw = cases[i]
        r, m, e, xf, so = _oracle(O, kw)
        assert stats[i]["steps"] == so["steps"], (i, kw)
        assert abs(stats[i]["dts_iters"] - so["dts_iters"]) <= stats[i]["margins"], (i, kw, stats[i], so)
        nc = kw["n"] + 1
        for got, ref in ((rho[i, :nc], r), (mom[i, :nc], m), (E[i, :nc], e)):
            assert _rel_l1(got.cpu().numpy(), ref) <= REL_L1, (i, kw)


def test_lax_warp_and_thread_loops_agree_bitwise(P):
    """dts_warp (lanes = cells, half warps = edges) and dts_thread (one thread) evaluate the same
    expressions in the same order: identical states and counts on every tab:iterations case."""
    cases = _cases()
    out = [P.lax_run([dict(c, dts_loop=loop) for c in cases]) for loop in (0, 1)]
    (r0, m0, e0, s0), (r1, m1, e1, s1) = out
    assert s0 == s1
    for a, b in ((r0, r1), (m0, m1), (e0, e1)):
        assert torch.equal(a, b)
