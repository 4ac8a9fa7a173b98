"""The seeded input generator (shared by both paths; no method arithmetic): SplitMix64 pinned
against a plain-integer re-implementation of the published constants, and the BASELINE recipe."""
import numpy as np

from paper_2211_00705_b200 import workloads as W

MASK = (1 << 64) - 1


def splitmix64_int(x):
    z = (x + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def u01_int(c, f, m, j):
    s = W.SEED
    for x in (c, f, m, j):
        s = splitmix64_int(s ^ x)
    return (s >> 11) * 2.0 ** -53


def test_splitmix_matches_integer_reference():
    for c, f, m, j in [(3, 0, 0, 0), (3, 1, 65535, 0), (5, 1, 0, 32767), (4, 0, 12345, 0)]:
        assert W.u01(c, f, m, j) == u01_int(c, f, m, j)
    # first value of the standard SplitMix64 sequence from state 0
    assert splitmix64_int(0) == 0xE220A8397B1DCDAF
    assert int(W.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_c3_recipe():
    w = W.c3(members=np.arange(2048))
    r = w["rho"][:, 0]
    assert r.min() >= 998 and r.max() <= 1002
    u = w["mom"][:, :1024] / w["rho"][:, :1024]
    assert np.all(u[:, 0] < 0) and np.all(u[:, -1] > 0)
    assert 20 <= np.abs(u).min() and np.abs(u).max() <= 200
    jumps = np.argmax(u > 0, axis=1)
    assert jumps.min() >= 0.3 * 1024 - 1 and jumps.max() <= 0.7 * 1024 + 1


def test_c4_recipe():
    w = W.c4(members=np.arange(512))
    r = w["rho"][:, 0]
    assert 0.015 <= r.min() and r.max() <= 0.03
    u = w["mom"][:, :4096] / w["rho"][:, :4096]
    assert np.all(u[:, :2048] > 0) and np.all(u[:, 2048:] < 0)


def test_c5_segments():
    rs, vs = W.c5_segments(n_cells=1 << 20)
    assert len(rs) == 256
    assert 999 <= rs.min() and rs.max() <= 1001 and -150 <= vs.min() and vs.max() <= 150
    rs2, vs2 = W.c5_segments(n_cells=1 << 20, first_segment=100, n_segments=10)
    np.testing.assert_array_equal(rs2, rs[100:110])
