"""Device CSR ingest (fglt_build_csr) == the host sanitiser == the reference's
build_adjacency contract (proj/src/graph.cpp:192-249): mirror, drop
self-loops, sort, dedupe, symmetry check, same error classes."""
import numpy as np
import pytest

from paper_2007_11111_b200 import _capi, graphs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = _capi.Context(0)
    yield c
    c.close()


def test_random_samples_match_host(ctx):
    rng = np.random.default_rng(3)
    for trial in range(20):
        n = int(rng.integers(1, 5000))
        ne = int(rng.integers(0, 20000))
        u = rng.integers(0, n, ne)
        v = rng.integers(0, n, ne)
        rp, ci, rep = ctx.build_csr(u, v, n)
        hrp, hci, hrep = graphs.csr_from_pairs(u, v, n)
        np.testing.assert_array_equal(rp, hrp)
        np.testing.assert_array_equal(ci, hci)
        assert rep == hrep


def test_rmat20_sample_matches_host(ctx):
    ne = graphs._lib().fglt_gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, None, None)
    u, v = graphs._two_pass(graphs._lib().fglt_gen_rmat, 20, 16, 0.57, 0.19, 0.19, 1)
    assert len(u) == ne
    rp, ci, _ = ctx.build_csr(u, v, 1 << 20)
    hrp, hci = graphs.rmat(20, 16, seed=1)
    np.testing.assert_array_equal(rp, hrp)
    np.testing.assert_array_equal(ci, hci)


def test_declared_n_and_empty(ctx):
    rp, ci, _ = ctx.build_csr(np.zeros(0, np.int64), np.zeros(0, np.int64), 7)
    assert rp.tolist() == [0] * 8 and len(ci) == 0
    rp, ci, _ = ctx.build_csr([0, 1], [1, 2], 10)
    assert len(rp) == 11 and ci.tolist() == [1, 0, 2, 1]


def test_sanitize_options_and_errors(ctx):
    with pytest.raises(_capi.TransformFailed) as e:
        ctx.build_csr([0], [1], 0, symmetrize=False)  # asymmetric
    assert e.value.code == 2
    rp, ci, _ = ctx.build_csr([0, 1], [1, 0], 0, symmetrize=False)
    assert ci.tolist() == [1, 0]
    with pytest.raises(_capi.TransformFailed) as e:
        ctx.build_csr([0, 2], [1, 2], 0, drop_self_loops=False)
    assert e.value.code == 2
    with pytest.raises(_capi.TransformFailed) as e:
        ctx.build_csr([0, 1], [1, 0], 0, dedupe=False)
    assert e.value.code == 2
    with pytest.raises(_capi.TransformFailed) as e:
        ctx.build_csr([-1], [1], 0)
    assert e.value.code == 2
    rp, ci, rep = ctx.build_csr([0, 1, 0, 2], [1, 0, 1, 2], 0)
    assert ci.tolist() == [1, 0] and rep == {"self_loops_dropped": 1, "duplicates_merged": 2}


def test_python_from_edges_uses_device_for_large_inputs():
    import paper_2007_11111_b200 as gt
    u, v = graphs._two_pass(graphs._lib().fglt_gen_rmat, 14, 16, 0.57, 0.19, 0.19, 9)
    g = gt.from_edges(np.stack([u, v], axis=1), n=1 << 14)
    hrp, hci, _ = graphs.csr_from_pairs(u, v, 1 << 14)
    assert g.num_vertices == len(hrp) - 1 and g.num_edges == len(hci) // 2
    for x in (0, 1, 77, 4096):
        assert g.neighbors(x) == hci[hrp[x]:hrp[x + 1]].tolist()
