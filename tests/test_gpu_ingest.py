"""Device CSR ingest (fglt_build_csr) == the UNMODIFIED reference
build_adjacency (proj/src/graph.cpp:192-249, oracle/_ref via
oracle.binding.ref_build_adjacency): same CSR, same BuildReport
(self_loops_dropped, duplicates_merged), same error class and message, for
symmetrize on/off, self-loops, duplicates and one-sided input."""
import numpy as np
import pytest

from oracle import binding as ob
from paper_2007_11111_b200 import _capi, graphs

pytestmark = pytest.mark.gpu

needs_ref = pytest.mark.skipif(not ob.have_ref(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ctx():
    c = _capi.Context(0)
    yield c
    c.close()


def both(ctx, u, v, n=0, **opt):
    """(device result or error, reference result or error), comparable."""
    try:
        rp, ci, rep = ctx.build_csr(u, v, n, **opt)
        dev = ("ok", rp.tolist(), ci.tolist(), rep["self_loops_dropped"], rep["duplicates_merged"])
    except _capi.TransformFailed as e:
        dev = ("err", e.code, e.msg)
    try:
        rp, ci, loops, dups = ob.ref_build_adjacency(u, v, n, **opt)
        ref = ("ok", rp.tolist(), ci.tolist(), loops, dups)
    except ob.OracleError as e:
        ref = ("err", e.code, e.msg)
    return dev, ref


@needs_ref
@pytest.mark.parametrize("symmetrize", [True, False])
def test_random_samples_match_reference(ctx, symmetrize):
    """Random pairs with self-loops and duplicates; with symmetrize off the
    samples are made symmetric by construction (plus duplicates) so both
    sides build a graph, and one-sided samples check the error path."""
    rng = np.random.default_rng(3 if symmetrize else 4)
    for trial in range(24):
        n = int(rng.integers(1, 3000))
        ne = int(rng.integers(0, 12000))
        u = rng.integers(0, n, ne)
        v = rng.integers(0, n, ne)
        if not symmetrize and trial % 3:
            u, v = np.concatenate([u, v, u[: ne // 4]]), np.concatenate([v, u, v[: ne // 4]])
        decl = n + int(rng.integers(0, 3)) if trial % 2 else 0
        dev, ref = both(ctx, u, v, decl, symmetrize=symmetrize)
        assert dev == ref, (trial, dev[:1], ref[:1], dev[-1:] if dev[0] == "err" else "", ref[-1:])


@needs_ref
def test_rmat20_sample_matches_reference(ctx):
    """16.8 M raw R-MAT samples (config 3's generator): the device CSR and
    report equal the reference's build_adjacency, and the CSR equals the
    workload generator's."""
    u, v = graphs._two_pass(graphs._lib().fglt_gen_rmat, 20, 16, 0.57, 0.19, 0.19, 1)
    rp, ci, rep = ctx.build_csr(u, v, 1 << 20)
    rrp, rci, loops, dups = ob.ref_build_adjacency(u, v, 1 << 20)
    np.testing.assert_array_equal(rp, rrp)
    np.testing.assert_array_equal(ci, rci)
    assert rep == {"self_loops_dropped": loops, "duplicates_merged": dups}
    hrp, hci = graphs.rmat(20, 16, seed=1)
    np.testing.assert_array_equal(rp, hrp)
    np.testing.assert_array_equal(ci, hci)


@needs_ref
@pytest.mark.parametrize("case", [
    # (u, v, declared_n, options)
    ([], [], 7, {}),
    ([0, 1], [1, 2], 10, {}),
    ([0], [1], 0, {"symmetrize": False}),                 # one-sided: odd entries
    ([0, 1, 2], [1, 2, 0], 0, {"symmetrize": False}),     # one-sided, even entries
    ([0, 1], [1, 0], 0, {"symmetrize": False}),
    ([0, 2, 5, 3], [1, 2, 5, 3], 0, {"drop_self_loops": False}),  # first loop in input order: 2
    ([0, 1], [1, 0], 0, {"dedupe": False}),
    ([-1], [1], 0, {}),
    ([0, 1, 0, 2], [1, 0, 1, 2], 0, {}),                  # reference test_smoke sanitisation
    ([0, 1, 0, 1], [1, 0, 1, 0], 0, {"symmetrize": False}),  # duplicates, symmetrize off
    ([3, 3], [3, 3], 0, {}),                              # only loops
])
def test_edge_cases_match_reference(ctx, case):
    u, v, n, opt = case
    dev, ref = both(ctx, np.array(u, np.int64), np.array(v, np.int64), n, **opt)
    assert dev == ref


def test_python_from_edges_is_device_ingest():
    """gt.from_edges goes through fglt_build_csr for every size (there is no
    host sort any more)."""
    import paper_2007_11111_b200 as gt
    u, v = graphs._two_pass(graphs._lib().fglt_gen_rmat, 14, 16, 0.57, 0.19, 0.19, 9)
    g = gt.from_edges(np.stack([u, v], axis=1), n=1 << 14)
    hrp, hci, _ = graphs.csr_from_pairs(u, v, 1 << 14)
    assert g.num_vertices == len(hrp) - 1 and g.num_edges == len(hci) // 2
    for x in (0, 1, 77, 4096):
        assert g.neighbors(x) == hci[hrp[x]:hrp[x + 1]].tolist()
    small = gt.from_edges([(0, 1), (1, 0), (0, 1), (2, 2)])
    assert small.num_vertices == 3 and small.num_edges == 1
