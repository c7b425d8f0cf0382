"""The reference's public per-kernel functions (proj/include/graphlet/
kernels.hpp:43-98; exercised by proj/tests/test_kernels.cpp) through the
graphlet:: C++ API on the device, bound as ``_core.kernels`` (additive).

Each function is compared against the oracle's per-kernel restatement
(oracle/fglt_oracle.c, pinned to the reference) on the Fig. 2 graph, small
structured graphs and seeded random families; caller-supplied vectors are
honoured literally (non-degree p1, perturbed C3), and the checked sites raise
CountOverflowError at the reference's graphlet id and vertex.
"""
import numpy as np
import pytest

import fglt_testutil as gu
import paper_2007_11111_b200 as gt
from oracle import binding as ob
from paper_2007_11111_b200 import _core, graphs

pytestmark = pytest.mark.gpu
K = _core.kernels
M64 = (1 << 64) - 1


def as_graph(rp, ci):
    rp = np.asarray(rp, np.int64)
    ci = np.asarray(ci, np.int64)
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = ci > rows
    e = np.stack([rows[keep], ci[keep]], axis=1)
    return gt.from_edges(e, n) if len(e) else gt.from_edges(np.zeros((0, 2), np.int64), n)


def cases():
    return {
        "demo": gu.demo(), "path5": gu.path(5), "cycle6": gu.cycle(6), "star5": gu.star(5),
        "k5": gu.complete(5), "k7": gu.complete(7), "tree30": gu.tree(30, 3),
        "er60": gu.er(60, 0.15, 4), "er300": gu.er(300, 0.05, 9), "reg": gu.regular(200, 7, 2),
        "rmat10": graphs.rmat(10, 8, seed=5), "rmat12": graphs.rmat(12, 16, seed=2),
    }


# numpy restatements of the checked kernels (python ints: exact) ------------
def d7_ref(rp, ci, p1):
    out = []
    for i in range(len(rp) - 1):
        acc = 0
        for j in ci[rp[i]:rp[i + 1]]:
            d = max(int(p1[j]) - 1, 0)
            c = d * (d - 1)
            if d >= 2 and c > M64:
                return ("err", 7, i)
            acc += c // 2 if d >= 2 else 0
            if acc > M64:
                return ("err", 7, i)
        out.append(acc)
    return np.array(out, np.uint64)


def d8_ref(p1):
    out = []
    for i, d in enumerate(int(x) for x in p1):
        if d < 3:
            out.append(0)
            continue
        x = ((d * (d - 1) // 2) & M64) * (d - 2)
        if x > M64:
            return ("err", 8, i)
        out.append(x // 3)
    return np.array(out, np.uint64)


def dip_ref(rp, ci, p1, c3, C3):
    n = len(rp) - 1
    d9, d10, d11 = [], [], []
    for i in range(n):
        nt = base = 0
        for e in range(rp[i], rp[i + 1]):
            j = ci[e]
            nt += int(c3[j])
            if nt > M64:
                return ("err", 9, i)
            t = int(C3[e]) * max(int(p1[j]) - 2, 0)
            if t > M64:
                return ("err", 10, i)
            base += t
            if base > M64:
                return ("err", 10, i)
        x11 = max(int(p1[i]) - 2, 0) * int(c3[i])
        if x11 > M64:
            return ("err", 11, i)
        d9.append(max(nt - ((2 * int(c3[i])) & M64), 0))
        d10.append(base)
        d11.append(x11)
    return tuple(np.array(x, np.uint64) for x in (d9, d10, d11))


def d13_ref(rp, ci, C3):
    n = len(rp) - 1
    out = np.zeros(n, np.uint64)
    for i in range(n):
        ni = set(ci[rp[i]:rp[i + 1]].tolist())
        tot = 0
        for j in ci[rp[i]:rp[i + 1]]:
            for b in range(rp[j], rp[j + 1]):
                if int(ci[b]) in ni:
                    tot += max(int(C3[b]) - 1, 0)
        out[i] = (tot & M64) // 2
    return out


# -------------------------------------------------------------------- tests
@pytest.mark.parametrize("name", list(cases()))
def test_per_kernel_functions_match_oracle(name):
    rp, ci = cases()[name]
    g = as_graph(rp, ci)
    v = ob.vectors(rp, ci)
    p1 = K.degree_vector(g)
    np.testing.assert_array_equal(p1, v["p1"])
    p2 = K.compute_p2(g, p1)
    np.testing.assert_array_equal(p2, v["p2"])
    c3, C3 = K.compute_c3_C3(g)
    np.testing.assert_array_equal(c3, v["c3"])
    np.testing.assert_array_equal(C3, v["C3"])
    np.testing.assert_array_equal(K.compute_p3(g, p1, p2, c3), v["p3"])
    c4, d14, touches = K.compute_c4_d14(g)
    np.testing.assert_array_equal(c4, v["c4"])
    np.testing.assert_array_equal(d14, v["d14"])
    assert touches == v["touches"]
    np.testing.assert_array_equal(K.compute_d13(g, C3), v["d13"])
    np.testing.assert_array_equal(K.compute_d15(g), ob.d15(rp, ci))
    np.testing.assert_array_equal(K.compute_d7(g, p1), d7_ref(rp, ci, p1))
    np.testing.assert_array_equal(K.compute_d8(p1), d8_ref(p1))
    for got, want in zip(K.compute_d9_d10_d11(g, p1, c3, C3), dip_ref(rp, ci, p1, c3, C3)):
        np.testing.assert_array_equal(got, want)


def test_fig2_known_answers():
    """The Fig. 2 graph's per-kernel columns equal the reference's own raw
    table (tests/fglt_testutil.py DEMO_RAW, proj/tests/testutil.hpp:40-62)."""
    rp, ci = gu.demo()
    g = as_graph(rp, ci)
    raw = gu.DEMO_RAW
    p1 = K.degree_vector(g)
    np.testing.assert_array_equal(K.compute_p2(g, p1), raw[:, 2])
    c3, C3 = K.compute_c3_C3(g)
    np.testing.assert_array_equal(c3, raw[:, 4])
    np.testing.assert_array_equal(K.compute_p3(g, p1, K.compute_p2(g, p1), c3), raw[:, 5])
    np.testing.assert_array_equal(K.compute_d7(g, p1), raw[:, 7])
    np.testing.assert_array_equal(K.compute_d8(p1), raw[:, 8])
    d9, d10, d11 = K.compute_d9_d10_d11(g, p1, c3, C3)
    np.testing.assert_array_equal(d9, raw[:, 9])
    np.testing.assert_array_equal(d10, raw[:, 10])
    np.testing.assert_array_equal(d11, raw[:, 11])
    c4, d14, _ = K.compute_c4_d14(g)
    np.testing.assert_array_equal(c4, raw[:, 12])
    np.testing.assert_array_equal(d14, raw[:, 14])
    np.testing.assert_array_equal(K.compute_d13(g, C3), raw[:, 13])
    np.testing.assert_array_equal(K.compute_d15(g), raw[:, 15])


def test_caller_vectors_are_used_as_given():
    """p1 need not be the degree vector and C3 need not be the graph's own:
    the reference computes with whatever it is handed."""
    rp, ci = gu.er(80, 0.12, 11)
    g = as_graph(rp, ci)
    rng = np.random.default_rng(5)
    n, nnz = len(rp) - 1, len(ci)
    p1 = rng.integers(0, 1000, n).astype(np.uint64)
    p2 = rng.integers(0, 1 << 40, n).astype(np.uint64)
    c3 = rng.integers(0, 50, n).astype(np.uint64)
    C3 = rng.integers(0, 9, nnz).astype(np.uint64)
    # p2 / p3 wrap and rectify exactly as the reference (unchecked)
    want_p2 = np.array([max(sum(int(p1[j]) for j in ci[rp[i]:rp[i + 1]]) - int(p1[i]), 0)
                        for i in range(n)], np.uint64)
    np.testing.assert_array_equal(K.compute_p2(g, p1), want_p2)
    walk = [sum(int(p2[j]) for j in ci[rp[i]:rp[i + 1]]) & M64 for i in range(n)]
    back = [(int(p1[i]) * max(int(p1[i]) - 1, 0) + 2 * int(c3[i])) & M64 for i in range(n)]
    np.testing.assert_array_equal(K.compute_p3(g, p1, p2, c3),
                                  np.array([max(a - b, 0) for a, b in zip(walk, back)], np.uint64))
    np.testing.assert_array_equal(K.compute_d7(g, p1), d7_ref(rp, ci, p1))
    for got, want in zip(K.compute_d9_d10_d11(g, p1, c3, C3), dip_ref(rp, ci, p1, c3, C3)):
        np.testing.assert_array_equal(got, want)
    # a C3 that is not the graph's own takes the literal (direct) d13 kernel
    np.testing.assert_array_equal(K.compute_d13(g, C3), d13_ref(rp, ci, C3))


def test_checked_sites_raise_at_reference_vertex():
    rp, ci = gu.demo()
    g = as_graph(rp, ci)
    n = len(rp) - 1
    big = np.full(n, 1 << 40, np.uint64)
    # choose3 of 2^40 overflows at the first vertex (graphlet 8)
    with pytest.raises(gt.CountOverflowError) as e:
        K.compute_d8(big)
    assert "graphlet 8" in str(e.value) and "vertex 0" in str(e.value)
    p1 = np.zeros(n, np.uint64)
    p1[3] = 1 << 33  # choose2(2^33 - 1) overflows for every neighbour of 3
    want = d7_ref(rp, ci, p1)
    assert want[0] == "err"
    with pytest.raises(gt.CountOverflowError) as e:
        K.compute_d7(g, p1)
    assert f"vertex {want[2]}" in str(e.value) and "graphlet 7" in str(e.value)
    # dipper: c3 sums overflow first (graphlet 9) at the lowest vertex
    c3 = np.full(n, 1 << 63, np.uint64)
    C3 = np.ones(len(ci), np.uint64)
    want = dip_ref(rp, ci, np.full(n, 3, np.uint64), c3, C3)
    assert want[0] == "err" and want[1] == 9
    with pytest.raises(gt.CountOverflowError) as e:
        K.compute_d9_d10_d11(g, np.full(n, 3, np.uint64), c3, C3)
    assert f"vertex {want[2]}" in str(e.value) and "graphlet 9" in str(e.value)
    # graphlet 10: the product C3 * (p1 - 2) overflows
    want = dip_ref(rp, ci, np.full(n, 1 << 40, np.uint64), np.zeros(n, np.uint64),
                   np.full(len(ci), 1 << 30, np.uint64))
    assert want[1] == 10
    with pytest.raises(gt.CountOverflowError) as e:
        K.compute_d9_d10_d11(g, np.full(n, 1 << 40, np.uint64), np.zeros(n, np.uint64),
                             np.full(len(ci), 1 << 30, np.uint64))
    assert f"vertex {want[2]}" in str(e.value) and "graphlet 10" in str(e.value)


def test_edgeless_and_empty():
    g = gt.from_edges(np.zeros((0, 2), np.int64), 7)
    p1 = K.degree_vector(g)
    assert (K.compute_p2(g, p1) == 0).all() and len(p1) == 7
    c3, C3 = K.compute_c3_C3(g)
    assert len(c3) == 7 and len(C3) == 0 and (c3 == 0).all()
    assert (K.compute_d13(g, C3) == 0).all()
    c4, d14, t = K.compute_c4_d14(g)
    assert (c4 == 0).all() and t == 0
    assert (K.compute_d15(g) == 0).all()
    assert len(K.compute_d8(np.zeros(0, np.uint64))) == 0
