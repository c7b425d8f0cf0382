"""The Python drop-in surface (paper_2007_11111_b200 == graphlet_transform).

Mirrors the reference's own smoke tests (proj/tests/python/test_smoke.py)
scenario by scenario. Host-only behaviour (graph building, parsing,
dictionaries, the conversion matrix) runs on CPU; anything that transforms is
marked gpu.
"""
import numpy as np
import pytest

import fglt_testutil as gu
import paper_2007_11111_b200 as gt


def demo_graph():
    """The Fig. 2 graph wrapped from its CSR (host only, no ingest)."""
    rp, ci = gu.demo()
    return gt.from_csr(rp, ci)


def test_graph_basics():
    g = demo_graph()
    assert g.num_vertices == 6
    assert g.num_edges == 9
    assert g.max_degree == 4
    assert sorted(g.neighbors(1)) == [0, 2, 3, 4]
    assert g.has_edge(0, 4) and not g.has_edge(0, 3)
    assert "n=6" in repr(g)


def test_from_csr_validates():
    with pytest.raises(gt.StructuralError):
        gt.from_csr([0, 1, 1], [1])            # asymmetric
    with pytest.raises(gt.StructuralError):
        gt.from_csr([0, 1], [0])               # self-loop
    g = gt.from_csr([0, 1], [0], validate=False)
    assert g.num_vertices == 1


@pytest.mark.gpu
def test_edges_as_array_equal_list():
    a = gt.from_edges(np.asarray(gu.DEMO_EDGES, dtype=np.int64))
    b = gt.from_edges(gu.DEMO_EDGES)
    assert (a.num_vertices, a.num_edges) == (b.num_vertices, b.num_edges)
    for v in range(6):
        assert a.neighbors(v) == b.neighbors(v) == demo_graph().neighbors(v)


@pytest.mark.gpu
def test_text_parsing_edge_list_and_mtx():
    text = "\n".join(f"{u} {v}" for (u, v) in gu.DEMO_EDGES)
    g = gt.from_text(text)
    assert g.num_vertices == 6 and g.num_edges == 9
    lines = ["%%MatrixMarket matrix coordinate pattern symmetric", "6 6 9"]
    lines += [f"{max(u, v) + 1} {min(u, v) + 1}" for (u, v) in gu.DEMO_EDGES]
    g2 = gt.from_text("\n".join(lines))
    assert g2.num_vertices == 6 and g2.num_edges == 9


@pytest.mark.gpu
def test_sanitization_and_errors():
    g = gt.from_edges([(0, 1), (1, 0), (0, 1), (2, 2)])
    assert g.num_vertices == 3 and g.num_edges == 1
    with pytest.raises(ValueError):
        gt.from_edges([(0, 1)], symmetrize=False)


def test_parse_and_dictionary_errors_host():
    with pytest.raises(ValueError):
        gt.from_text("0 x")
    with pytest.raises(gt.ParseError):
        gt.graphlet_ids("99")
    with pytest.raises(gt.ParseError):
        gt.graphlet_ids("4-2")
    with pytest.raises(gt.ParseError):
        gt.graphlet_ids("1,")


def test_oracle_tables_host():
    """The brute-force oracle (host, csrc/brute.cpp) reproduces the Fig. 2
    tables and equals the reference's own oracle on random graphs."""
    g = demo_graph()
    np.testing.assert_array_equal(gt.oracle_raw(g), gu.DEMO_RAW)
    np.testing.assert_array_equal(gt.oracle_net(g), gu.DEMO_NET)
    with pytest.raises(gt.StructuralError):
        gt.oracle_raw(g, cap=5)
    from oracle import binding as ob
    if not ob.have_ref():
        pytest.skip("oracle/_ref not built")
    for t in range(40):
        n = 3 + t % 30
        rp, ci = ob.ref_er_graph(n, (0.1, 0.25, 0.5)[t % 3], 77 + t)
        h = gt.from_csr(rp, ci)
        rraw, rnet = ob.ref_oracle(rp, ci)
        np.testing.assert_array_equal(gt.oracle_raw(h), rraw)
        np.testing.assert_array_equal(gt.oracle_net(h), rnet)


SPECS = ["all", " all ", "0-4", " 0-4 ", "4,15", " 2, 5-7 ", "15", "0", "1", "3-3",
         "1,", "1, ", ",1", ",", "-3", "3-", "4-2", "x", "16", "0-16", "", "   ", "1,,2",
         "2 ,3", "2- 5", "+3", "07", "1-1,1", "12,14,13"]


@pytest.mark.parametrize("spec", SPECS)
def test_dictionary_grammar_matches_reference(spec):
    """Every spec: the same ids, implicitly added ids, or error message as
    the UNMODIFIED reference parse_dictionary (oracle/_ref)."""
    from oracle import binding as ob
    if not ob.have_ref():
        pytest.skip("oracle/_ref not built")
    try:
        want = ob.ref_parse_dictionary(spec)
    except ValueError as e:
        with pytest.raises(gt.ParseError) as got:
            gt.graphlet_ids(spec)
        assert str(got.value) == str(e)
        return
    assert gt.graphlet_ids(spec) == want[0]


def test_dictionary_specs():
    assert gt.graphlet_ids("0-4") == [0, 1, 2, 3, 4]
    assert gt.graphlet_ids("4,15") == [0, 1, 4, 15]
    assert gt.graphlet_ids(" 2, 5-7 ") == [0, 1, 2, 5, 6, 7]
    assert gt.graphlet_ids("all") == list(range(16))


def test_conversion_matrix_host():
    u = gt.conversion_matrix("all")
    assert u.shape == (16, 16) and u.dtype == np.uint64
    assert u[2, 4] == 2 and u[5, 15] == 6 and u[13, 14] == 0
    assert (np.tril(u, -1) == 0).all() and (np.diag(u) == 1).all()
    s = gt.conversion_matrix("0,1,5,9,13")
    assert s[2, 4] == 4 and s[2, 3] == 2 and s[3, 4] == 2


def test_graphlet_names():
    names = gt.graphlet_names()
    assert len(names) == 16
    assert names[0] == "singleton"
    assert "claw" in names[8]


@pytest.mark.gpu
def test_cross_check_legs():
    ok, report = gt.cross_check(demo_graph())
    assert ok and "all legs pass" in report, report


@pytest.mark.gpu
def test_transform_matches_reference_tables():
    raw, net = gt.transform(demo_graph())
    np.testing.assert_array_equal(raw, gu.DEMO_RAW)
    np.testing.assert_array_equal(net, gu.DEMO_NET)


@pytest.mark.gpu
def test_sub_dictionary_columns():
    g = demo_graph()
    raw = gt.raw_frequencies(g, dict="0-4")
    np.testing.assert_array_equal(raw, gu.DEMO_RAW[:, :5])
    raw_with_closure = gt.raw_frequencies(g, dict="4,15")
    np.testing.assert_array_equal(raw_with_closure, gu.DEMO_RAW[:, [0, 1, 4, 15]])


@pytest.mark.gpu
def test_conversion_matrix_round_trip():
    g = demo_graph()
    u = gt.conversion_matrix("all")
    raw, net = gt.transform(g)
    np.testing.assert_array_equal(net @ u.T, raw)


@pytest.mark.gpu
def test_text_parsing_transform_equal():
    text = "\n".join(f"{u} {v}" for (u, v) in gu.DEMO_EDGES)
    lines = ["%%MatrixMarket matrix coordinate pattern symmetric", "6 6 9"]
    lines += [f"{max(u, v) + 1} {min(u, v) + 1}" for (u, v) in gu.DEMO_EDGES]
    raw1, _ = gt.transform(gt.from_text(text))
    raw2, _ = gt.transform(gt.from_text("\n".join(lines)))
    np.testing.assert_array_equal(raw1, raw2)


@pytest.mark.gpu
def test_bad_dictionary_raises():
    with pytest.raises(ValueError):
        gt.raw_frequencies(demo_graph(), dict="99")


@pytest.mark.gpu
def test_lenient_flag():
    k4 = gt.from_edges([(u, v) for u in range(4) for v in range(u + 1, 4)])
    with pytest.raises(ValueError):
        gt.transform(k4, dict="5,13")
    with pytest.raises(gt.InconsistencyError):
        gt.transform(k4, dict="5,13")
    raw, net = gt.transform(k4, dict="5,13", lenient=True)
    assert net[:, 2].tolist() == [0, 0, 0, 0]


@pytest.mark.gpu
def test_overflow_maps_to_overflow_error():
    leaves = 1 << 22
    edges = np.stack([np.zeros(leaves, np.int64), np.arange(1, leaves + 1)], axis=1)
    star = gt.from_edges(edges)
    with pytest.raises(OverflowError):
        gt.transform(star, dict="8")


@pytest.mark.gpu
def test_results_own_their_memory():
    g = demo_graph()
    raw, net = gt.transform(g)
    del g
    assert raw.flags["OWNDATA"] is False  # numpy views the device-filled table
    np.testing.assert_array_equal(raw, gu.DEMO_RAW)


@pytest.mark.gpu
def test_matches_oracle_random_family():
    from oracle import binding as ob
    rng = np.random.default_rng(20260811)
    for trial in range(12):
        n = int(rng.integers(10, 60))
        edges = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.2]
        g = gt.from_edges(edges, n=n)
        rp, ci = gu.from_pairs(edges, n)
        raw, net = gt.transform(g)
        oraw, onet = ob.transform(rp, ci)
        np.testing.assert_array_equal(raw, oraw)
        np.testing.assert_array_equal(net, onet)
