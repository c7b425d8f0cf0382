"""GPU parity through the C-ABI (libfglt.so) against the pinned oracle.

Bit-exact for every raw and net entry (integer work). Cases follow the
reference's own tests: Fig. 2 golden tables (proj/tests/testutil.hpp:40-62),
sub-dictionaries (acceptance.cpp:74-93), the 208-graph oracle family
(acceptance.cpp:114-146), edge cases (edgeless graph test_kernels.cpp:229-238,
incomplete family test_pipeline.cpp:55-65, corrupted raw
test_conversion.cpp:63-76), and the synthetic configs at sizes the oracle
finishes in seconds.
"""
import os

import numpy as np
import pytest

from oracle import binding as ob
from paper_2007_11111_b200 import _capi, graphs
import fglt_testutil as gu

pytestmark = pytest.mark.gpu

FULL = 0xFFFF
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctx():
    c = _capi.Context(0)
    yield c
    c.close()


def check_same(ctx, rp, ci, mask=FULL, lenient=False, d15_mode=0):
    raw, net, st = ctx.transform_host(rp, ci, mask, lenient)
    oraw, onet = ob.transform(rp, ci, mask, lenient, d15_mode)
    assert raw.shape == oraw.shape
    bad = np.argwhere(raw != oraw)
    assert len(bad) == 0, f"raw differs at {bad[:5]}: gpu {raw[tuple(bad[0])]} oracle {oraw[tuple(bad[0])]}"
    bad = np.argwhere(net != onet)
    assert len(bad) == 0, f"net differs at {bad[:5]}"
    return raw, net, st


def test_fig2_golden_tables(ctx):
    rp, ci = gu.demo()
    raw, net, st = ctx.transform_host(rp, ci)
    np.testing.assert_array_equal(raw, gu.DEMO_RAW)
    np.testing.assert_array_equal(net, gu.DEMO_NET)
    assert st["kernel_launches"] > 0


@pytest.mark.parametrize("ids", [[0, 1], [0, 1, 2, 3, 4], [0, 1, 12], [0, 1, 4, 15]])
def test_fig2_sub_dictionaries(ctx, ids):
    rp, ci = gu.demo()
    mask = _capi.dict_mask(ids)
    raw, net, _ = ctx.transform_host(rp, ci, mask)
    full_ids = _capi.mask_ids(mask)
    np.testing.assert_array_equal(raw, gu.DEMO_RAW[:, full_ids])
    # acceptance.cpp:84-93: {0,1,12} has an identity conversion
    want = gu.DEMO_RAW if ids == [0, 1, 12] else gu.DEMO_NET
    np.testing.assert_array_equal(net, want[:, full_ids])


def test_config1_parity(ctx):
    rp, ci = graphs.er(2000, 0.004, 1)
    raw, net, st = check_same(ctx, rp, ci)
    # SURVEY App. B column sums (reference-produced)
    assert raw.sum(0).tolist() == [2000, 16212, 132038, 66019, 243, 1074176, 1074176, 538500,
                                   179500, 2014, 4028, 2014, 2240, 2, 2, 0]
    assert st["p2_row_touches"] == st["W"] - 16212


def test_oracle_family_208(ctx):
    """The acceptance family: 120 ER, 60 regular, 10 trees, K2-K6, C3-C8, stars."""
    seed = 0x51AB5EED
    cases = []
    for i in range(120):
        n = 5 + (i * 7) % 36
        p = 0.1 if i % 3 == 0 else 0.2 if i % 3 == 1 else 0.4
        cases.append(gu.er(n, p, seed + i))
    for d in (3, 4, 5):
        for j in range(20):
            n = 6 + 2 * (j % 18)
            cases.append(gu.regular(n, d, seed + 1000 + j + d))
    for n in (2, 5, 9, 14, 20, 27, 33, 40, 15, 25):
        cases.append(gu.tree(n, seed + 31 * n))
    cases += [gu.complete(n) for n in range(2, 7)]
    cases += [gu.cycle(n) for n in range(3, 9)]
    cases += [gu.star(k) for k in range(2, 9)]
    for rp, ci in cases:
        check_same(ctx, rp, ci)


def test_dense_small_graphs(ctx):
    for n in (4, 5, 8, 12, 20, 33, 64):
        check_same(ctx, *gu.complete(n))
    for seed in range(6):
        check_same(ctx, *gu.er(60, 0.5, 100 + seed))
        check_same(ctx, *gu.er(200, 0.2, 200 + seed))


def test_edgeless_and_empty(ctx):
    rp = np.zeros(5, np.int32)
    ci = np.zeros(0, np.int32)
    raw, net, _ = ctx.transform_host(rp, ci)
    assert (raw[:, 0] == 1).all() and (raw[:, 1:] == 0).all()
    assert (net == raw).all()
    raw, net, _ = ctx.transform_host(np.zeros(1, np.int32), ci)
    assert raw.shape == (0, 16)
    # isolated vertices mixed in
    check_same(ctx, *gu.from_pairs([(0, 5), (5, 9), (9, 0), (9, 12)], 20))


def test_random_subdicts_and_lenient(ctx):
    rng = np.random.default_rng(20260811)
    for trial in range(120):
        n = int(rng.integers(2, 45))
        rp, ci = gu.er(n, float(rng.choice([0.1, 0.3, 0.6])), int(rng.integers(1 << 30)))
        mask = int(rng.integers(0, 1 << 16))
        lenient = bool(trial % 2)
        try:
            oraw, onet = ob.transform(rp, ci, mask, lenient)
            oerr = None
        except ob.OracleError as e:
            oerr = (e.code, e.graphlet_id, e.vertex)
        try:
            raw, net, _ = ctx.transform_host(rp, ci, mask, lenient)
            gerr = None
        except _capi.TransformFailed as e:
            gerr = (e.code, e.graphlet_id, e.vertex)
        assert gerr == oerr
        if oerr is None:
            np.testing.assert_array_equal(raw, oraw)
            np.testing.assert_array_equal(net, onet)


def test_incomplete_family_inconsistency(ctx):
    """test_pipeline.cpp:55-65 / test_smoke.py:125-130."""
    rp, ci = gu.complete(4)
    mask = _capi.dict_mask([5, 13])
    with pytest.raises(_capi.TransformFailed) as ei:
        ctx.transform_host(rp, ci, mask)
    assert ei.value.code == 4
    raw, net, _ = ctx.transform_host(rp, ci, mask, lenient=True)
    assert net[:, 2].tolist() == [0, 0, 0, 0]


def test_net_from_raw_corrupted(ctx):
    """test_conversion.cpp:63-76: raw(0,15)+1 -> InconsistencyError(vertex 0, graphlet 14)."""
    rp, ci = gu.demo()
    raw, _, _ = ctx.transform_host(rp, ci)
    raw[0, 15] += 1
    with pytest.raises(_capi.TransformFailed) as ei:
        ctx.net_from_raw(raw, FULL)
    assert (ei.value.code, ei.value.vertex, ei.value.graphlet_id) == (4, 0, 14)
    net = ctx.net_from_raw(raw, FULL, lenient=True)
    assert net[0, 14] == 0


def test_net_from_raw_custom_matrix(ctx):
    """net_from_raw honours the caller's ConversionMatrix (conversion.hpp:
    14-37,49-51), not the built-in U16(s,s): a modified unit upper-triangular
    U gives exactly the back substitution of that U (Python integers)."""
    rp, ci = gu.er(40, 0.3, 77)
    mask = FULL
    raw, net16, _ = ctx.transform_host(rp, ci, mask)
    U = ob.u16().astype(np.uint64)
    np.testing.assert_array_equal(ctx.net_from_raw(raw, mask, U=U), net16)
    U2 = U.copy()
    U2[2, 4] = 1          # was 2
    U2[5, 15] = 5         # was 6
    got = ctx.net_from_raw(raw, mask, lenient=True, U=U2)
    for v in range(raw.shape[0]):
        x = [0] * 16
        for r in range(15, -1, -1):
            a = sum(int(U2[r, c]) * x[c] for c in range(r + 1, 16))
            x[r] = max(int(raw[v, r]) - a, 0)
        assert got[v].tolist() == x
    bad = U2.copy()
    bad[3, 1] = 1  # below the diagonal
    with pytest.raises(_capi.TransformFailed) as ei:
        ctx.net_from_raw(raw, mask, U=bad)
    assert ei.value.code == 2


def test_choose3_overflow_site(ctx):
    """choose3 (col 8) is the one checked site reachable with int32 CSR:
    a star with 2^22 leaves overflows d(d-1)/2*(d-2). Reference order: the
    col-8 fill raises OverflowError(graphlet 8, vertex 0)."""
    leaves = 1 << 22
    rp = np.zeros(leaves + 2, np.int64)
    rp[1] = leaves
    rp[2:] = leaves + np.arange(1, leaves + 1)
    ci = np.concatenate([np.arange(1, leaves + 1), np.zeros(leaves, np.int64)])
    mask = _capi.dict_mask([8])
    with pytest.raises(_capi.TransformFailed) as ei:
        ctx.transform_host(rp.astype(np.int32), ci.astype(np.int32), mask)
    assert (ei.value.code, ei.value.graphlet_id, ei.value.vertex) == (3, 8, 0)


@pytest.mark.parametrize("scale", [10, 12, 13])
def test_rmat_parity(ctx, scale):
    rp, ci = graphs.rmat(scale, 16, seed=scale)
    check_same(ctx, rp, ci, d15_mode=1)


def test_sbm_rgg_parity(ctx):
    check_same(ctx, *graphs.sbm(512, 64, 0.3, 3.0, 5), d15_mode=1)
    check_same(ctx, *graphs.rgg(50000, 3.0, 2), d15_mode=1)
    check_same(ctx, *graphs.rgg(20000, 12.0, 9), d15_mode=1)


def test_permutation_equivariance(ctx):
    rng = np.random.default_rng(808)
    for trial in range(5):
        rp, ci = gu.er(300, 0.05, 1000 + trial)
        pi = rng.permutation(300)
        rp2, ci2 = gu.permute(rp, ci, pi)
        a, _, _ = ctx.transform_host(rp, ci)
        b, _, _ = ctx.transform_host(rp2, ci2)
        np.testing.assert_array_equal(a, b[pi])


def test_determinism_repeat(ctx):
    rp, ci = graphs.rmat(14, 16, seed=7)
    a = ctx.transform_host(rp, ci)
    b = ctx.transform_host(rp, ci)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_one_shot_entry_point():
    rp, ci = gu.demo()
    raw, net, _ = _capi.transform(rp, ci)
    np.testing.assert_array_equal(raw, gu.DEMO_RAW)
    np.testing.assert_array_equal(net, gu.DEMO_NET)


FORCED = [
    ("c4 hash P=1", _capi.DEBUG_C4_CLASS, 2, 1),
    ("c4 hash P=3", _capi.DEBUG_C4_CLASS, 2, 3),
    ("c4 packed tiles", _capi.DEBUG_C4_CLASS, 3, 0),
    ("c4 32-bit tiles", _capi.DEBUG_C4_CLASS, 4, 0),
    ("c4 small packed tiles", _capi.DEBUG_C4_CLASS, 5, 0),
    ("roots bin 1", _capi.DEBUG_ROOTS_BIN, 1, 0),
    ("roots bin 2", _capi.DEBUG_ROOTS_BIN, 2, 0),
    ("roots bin 4", _capi.DEBUG_ROOTS_BIN, 4, 0),
    ("roots global slab", _capi.DEBUG_ROOTS_BIN, 5, 0),
]


@pytest.mark.parametrize("label,key,value,parts", FORCED, ids=[f[0] for f in FORCED])
def test_forced_code_paths(label, key, value, parts):
    """Every internal path (normally reached only at scale) must give the
    same bits: force it for all roots on small graphs."""
    c = _capi.Context(0)
    c.set_debug(key, value)
    if parts:
        c.set_debug(_capi.DEBUG_C4_PARTS, parts)
    cases = [gu.er(200, 0.2, 7), gu.complete(40), graphs.rmat(12, 16, seed=5),
             graphs.sbm(64, 64, 0.3, 3.0, 9), gu.star(70), gu.demo()]
    for rp, ci in cases:
        check_same(c, rp, ci, d15_mode=1)
    c.close()


def test_relabel_paths_agree():
    """Low-degree graphs build their relabelled rows with the in-register row
    sort (k_fill_sort: every lanes-per-row / elements-per-lane shape below);
    forcing the global transpose sort must give the same bits."""
    cases = [gu.regular(400, 4, 11), gu.er(2000, 0.004, 1), gu.er(500, 0.02, 3),
             gu.er(300, 0.06, 5), graphs.sbm(64, 64, 0.3, 3.0, 9), gu.er(200, 0.3, 2),
             gu.star(70), gu.complete(40), gu.demo()]
    c = _capi.Context(0)
    f = _capi.Context(0)
    f.set_debug(_capi.DEBUG_ROW_SORT, 2)
    for rp, ci in cases:
        check_same(c, rp, ci, d15_mode=1)
        a = c.transform_host(rp, ci)
        b = f.transform_host(rp, ci)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
    c.close()
    f.close()


@pytest.mark.parametrize("flat", [0, 64, 255])
@pytest.mark.parametrize("c4class", [0, 2, 3, 4, 5])
def test_vertex_order_paths_agree(flat, c4class):
    """Graphs with d_max <= the flat threshold keep the caller's vertex order
    among active vertices (k_degree_keys; dense 4-cycle counters then use one
    8-bit band); threshold 0 always relabels by degree. Same bits either way,
    under every forced 4-cycle class."""
    c = _capi.Context(0)
    c.set_debug(_capi.DEBUG_FLAT_DMAX, flat)
    c.set_debug(_capi.DEBUG_C4_CLASS, c4class)
    cases = [gu.regular(400, 4, 11), gu.er(2000, 0.004, 1), gu.er(300, 0.06, 5),
             graphs.sbm(64, 64, 0.3, 3.0, 9), gu.er(200, 0.3, 2), gu.star(70),
             gu.complete(40), gu.complete(17), graphs.rmat(11, 8, seed=3), gu.demo()]
    for rp, ci in cases:
        check_same(c, rp, ci, d15_mode=1)
    c.close()


@pytest.mark.parametrize("hub", [1, 2])
@pytest.mark.parametrize("rbin", [0, 1, 3, 5])
def test_hub_rows_paths(hub, rbin):
    """Hub-row pair checks (forced for every hub member) and the pure probe
    path (hub rows off) must give the same bits, in every block bin."""
    c = _capi.Context(0)
    c.set_debug(_capi.DEBUG_HUB, hub)
    c.set_debug(_capi.DEBUG_ROOTS_BIN, rbin)
    cases = [gu.er(300, 0.15, 11), gu.complete(48), graphs.rmat(12, 16, seed=6),
             graphs.sbm(64, 64, 0.3, 3.0, 4), gu.star(90), gu.demo()]
    for rp, ci in cases:
        check_same(c, rp, ci, d15_mode=1)
    c.close()


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("rbin", [0, 2, 5])
def test_triangle_list_paths(mode, rbin):
    """Diamonds from the triangle list (auto), without it (1), and with a pool
    so small that most roots fall back to the probing pass mid-list (2) give
    the same bits, in every block bin and with hub-row pair checks forced."""
    c = _capi.Context(0)
    c.set_debug(_capi.DEBUG_TRILIST, mode)
    c.set_debug(_capi.DEBUG_ROOTS_BIN, rbin)
    c.set_debug(_capi.DEBUG_HUB, 2)
    cases = [gu.er(300, 0.15, 11), gu.complete(48), graphs.rmat(12, 16, seed=6),
             graphs.sbm(64, 64, 0.3, 3.0, 4), gu.star(90), gu.demo()]
    for rp, ci in cases:
        check_same(c, rp, ci, d15_mode=1)
    c.close()


def test_repeat_determinism_at_scale():
    """Bit-identical results across repeated runs at a size where every
    root bin and 4-cycle class is populated (guards against lost updates;
    a 64-bit shared atomicAdd once dropped d13 contributions here)."""
    rp, ci = graphs.rmat(19, 16, seed=3)
    c = _capi.Context(0)
    base = c.transform_host(rp, ci)
    for _ in range(6):
        raw, net, _ = c.transform_host(rp, ci)
        np.testing.assert_array_equal(raw, base[0])
        np.testing.assert_array_equal(net, base[1])
    c.close()


def test_reference_golden_fixtures(ctx):
    """Tables produced by the reference itself (tests/golden/make_golden.py)."""
    import hashlib
    import json
    import os
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    cfg = json.load(open(os.path.join(gold, "config1.json")))
    rp, ci = graphs.er(2000, 0.004, 1)
    raw, net, _ = ctx.transform_host(rp, ci)
    assert hashlib.sha256(raw.tobytes()).hexdigest() == cfg["raw_sha256"]
    assert hashlib.sha256(net.tobytes()).hexdigest() == cfg["net_sha256"]
    z = np.load(os.path.join(gold, "small_tables.npz"))
    for name in sorted({k[:-3] for k in z.files if k.endswith("_rp")}):
        raw, net, _ = ctx.transform_host(z[name + "_rp"], z[name + "_ci"])
        np.testing.assert_array_equal(raw, z[name + "_raw"], err_msg=name)
        np.testing.assert_array_equal(net, z[name + "_net"], err_msg=name)
    rp, ci = z["rmat10_rp"], z["rmat10_ci"]
    for key in z.files:
        if not key.startswith("rmat10_m"):
            continue
        mask, lenient = int(key[8:12], 16), bool(int(key[14]))
        fresh = _capi.Context(0)  # a first call on a fresh context must be right too
        if key.endswith("_err"):
            with pytest.raises(_capi.TransformFailed) as ei:
                fresh.transform_host(rp, ci, mask, lenient)
            assert [ei.value.code, ei.value.graphlet_id, ei.value.vertex] == z[key].tolist()
        elif key.endswith("_raw"):
            raw, net, _ = fresh.transform_host(rp, ci, mask, lenient)
            np.testing.assert_array_equal(raw, z[key])
            np.testing.assert_array_equal(net, z[key[:-4] + "_net"])


def test_stats_contract(ctx):
    """Step names in reference plan order (test_pipeline.cpp:78-94) and the
    touch identity / bound (test_pipeline.cpp:96-108)."""
    rp, ci = gu.demo()
    _, _, st = ctx.transform_host(rp, ci, _capi.dict_mask([]), timings=True)
    assert [k for k, _ in st["kernel_times"]] == ["degrees", "column fill", "conversion"]
    _, _, st = ctx.transform_host(rp, ci, _capi.dict_mask([12]), timings=True)
    assert [k for k, _ in st["kernel_times"]] == ["degrees", "four-cycle rows", "column fill",
                                                  "conversion"]
    _, _, st = ctx.transform_host(rp, ci, 0xFFFF, timings=True)
    assert [k for k, _ in st["kernel_times"]] == [
        "degrees", "triangles", "two-paths", "three-paths", "four-cycle rows", "diamond rows",
        "tetrahedra", "column fill", "conversion"]
    rp, ci = gu.regular(400, 4, 11)
    _, _, st = ctx.transform_host(rp, ci)
    assert 0 < st["p2_row_touches"] <= st["p2_touch_bound"]
    assert st["p2_row_touches"] == st["W"] - len(ci)


def test_per_call_scratch_and_phases(ctx):
    """TransformStats are per call (the reference resets its MemoryTracker
    each call, kernels.cpp:312): a small graph after a large one reports the
    small graph's scratch and launches; the scratch report lists exactly the
    counted buffers; phases carry CUDA-event times and the dense wedge units."""
    big_rp, big_ci = graphs.rmat(14, 16, seed=2)
    _, _, st_big = ctx.transform_host(big_rp, big_ci, timings=True)
    rp, ci = gu.regular(400, 4, 11)
    _, _, st = ctx.transform_host(rp, ci)
    assert 0 < st["peak_aux_words"] < st_big["peak_aux_words"]
    assert 0 < st["kernel_launches"] < 200
    rep = ctx.scratch_report()
    counted = sum(b for b, staging in rep.values() if not staging)
    assert counted // 8 == st["peak_aux_words"]
    assert st["largest_aux_alloc_words"] < (400 * 400) // 8
    names = [p[0] for p in st_big["phases"]]
    for must in ("prepare", "triangle pass", "four-cycle rows", "column fill"):
        assert must in names
    assert all(secs >= 0 for _, secs, _ in st_big["phases"])
    assert ctx.smem_atomic_rate() > 1e11


def test_sharded_stages_byte_identical(ctx):
    """The staged (multi-rank) decomposition run rank by rank on one GPU:
    partial edge counts and root vectors summed across 'ranks' give the same
    bytes as the single-call path (the NCCL exchange is a plain integer sum)."""
    import torch
    from paper_2007_11111_b200.dist import CudaStages
    rp, ci = graphs.rmat(14, 16, seed=4)
    n, nnz = len(rp) - 1, len(ci)
    want_raw, want_net, _ = ctx.transform_host(rp, ci)
    dev = torch.device("cuda", 0)
    rp_d, ci_d = torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev)
    for world in (2, 3, 8):
        st = CudaStages(dev)
        st.prepare(rp_d, ci_d, n, nnz, 0xFFFF, False)
        b = st.bounds(world)
        assert b[0] == 0 and b[-1] == n and (np.diff(b) >= 0).all()
        c3 = None
        for r in range(world):
            part = st.triangles(int(b[r]), int(b[r + 1])).clone()
            c3 = part if c3 is None else c3 + part
        st.triangles(0, 0).copy_(c3)
        st.local()
        vec = None
        for r in range(world):
            part = st.roots(int(b[r]), int(b[r + 1])).clone()
            st.roots(0, 0).zero_()
            vec = part if vec is None else vec + part
        st.roots(0, 0).copy_(vec)
        raw = torch.empty((n, 16), dtype=torch.int64, device=dev)
        net = torch.empty((n, 16), dtype=torch.int64, device=dev)
        rc, err = st.epilogue(0, n, raw, net)
        assert rc == 0, err
        np.testing.assert_array_equal(raw.cpu().numpy().view(np.uint64), want_raw)
        np.testing.assert_array_equal(net.cpu().numpy().view(np.uint64), want_net)


@pytest.mark.parametrize("cfg", [2, 5, 3])
def test_full_size_config_parity(ctx, cfg):
    """BASELINE.json configs 2 (RGG 2M), 5 (SBM 4.2M) and 3 (R-MAT scale 20)
    at full size, every raw and net entry against the oracle (d15 by the
    oriented K4 counter, pinned to the reference's compute_d15)."""
    name, rp, ci = graphs.config(cfg)
    raw, net, _ = ctx.transform_host(rp, ci)
    oraw, onet = ob.transform(rp, ci, FULL, False, 1)
    assert np.array_equal(raw, oraw), name
    assert np.array_equal(net, onet), name


@pytest.mark.gpu
def test_bench_two_ranks_gloo():
    """bench.py's N>1 code path (CSR broadcast, root blocks, the two
    all-reduces, row gather, max-over-ranks timing) end to end under torchrun
    with world size 2. Only one GPU exists here, so both ranks share it over
    gloo (host-staged collectives; no rank's kernels wait on the other's); on
    the 8-GPU box the same code runs over NCCL."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, FGLT_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--config", "1", "--verify"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0 and rec["e2e"]["value"] > 0


def test_config4_full_size_properties():
    """BASELINE.json config 4 (R-MAT scale 23, 129M edges) at full size. The
    oracle's full transform is out of reach here (its reference-algorithm
    4-cycle and diamond passes are O(W) random accesses, W = 1.34e12), so:
    (1) the O(nnz) sub-dictionary {0,1,2,3,7,8} raw AND net against the
    oracle, bit for bit; (2) the full Sigma16 tables are byte-identical to the
    staged 8-rank decomposition (different root partition, list pools and
    schedules); (3) raw = U net exactly for every vertex (the conversion leg);
    (4) degree-sum identities of columns 1 and 3."""
    import torch
    from paper_2007_11111_b200.dist import CudaStages
    name, rp, ci = graphs.config(4)
    n, nnz = len(rp) - 1, len(ci)
    cheap = _capi.dict_mask([2, 3, 7, 8])
    ctx = _capi.Context(0)
    raw_c, net_c, _ = ctx.transform_host(rp, ci, cheap)
    oraw, onet = ob.transform(rp, ci, cheap, False, 0)
    assert np.array_equal(raw_c, oraw) and np.array_equal(net_c, onet), name
    raw, net, _ = ctx.transform_host(rp, ci)
    ctx.close()  # its workspace (triangle-list pool included) goes back before (2)
    assert np.array_equal(raw[:, [0, 1, 2, 3, 7, 8]], oraw)
    assert int(raw[:, 1].sum()) == nnz
    deg = np.diff(rp).astype(np.uint64)
    assert np.array_equal(raw[:, 3], deg * (deg - 1) // 2)
    # (3) raw = U net, exact in uint64 (no wrap: every term is <= raw)
    U = ob.u16()
    back = net.copy()
    for r in range(16):
        for c in range(r + 1, 16):
            if U[r, c]:
                back[:, r] += U[r, c] * net[:, c]
    assert np.array_equal(back, raw)
    assert (net <= raw).all()
    # (2) staged 8-rank decomposition on one device, byte identical
    dev = torch.device("cuda", 0)
    rp_d, ci_d = torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev)
    world = 8
    st = CudaStages(dev)
    st.prepare(rp_d, ci_d, n, nnz, 0xFFFF, False)
    b = st.bounds(world)
    c3 = view = None
    for r in range(world):
        view = st.triangles(int(b[r]), int(b[r + 1]))  # aliases the context's edge counts
        c3 = view.clone() if c3 is None else c3 + view
    view.copy_(c3)
    st.local()
    vec = None
    for r in range(world):
        view = st.roots(int(b[r]), int(b[r + 1]))  # aliases the context's vectors
        vec = view.clone() if vec is None else vec + view
        view.zero_()
    view.copy_(vec)
    del c3, vec, rp_d, ci_d
    raw_d = torch.empty((n, 16), dtype=torch.int64, device=dev)
    net_d = torch.empty((n, 16), dtype=torch.int64, device=dev)
    rc, err = st.epilogue(0, n, raw_d, net_d)
    assert rc == 0, err
    assert np.array_equal(raw_d.cpu().numpy().view(np.uint64), raw)
    assert np.array_equal(net_d.cpu().numpy().view(np.uint64), net)


def test_release_workspace_then_transform():
    """Freeing the kept workspace between calls changes nothing but memory."""
    import paper_2007_11111_b200 as gt
    rp, ci = graphs.rmat(12, 16, seed=8)
    c = _capi.Context(0)
    a = c.transform_host(rp, ci)
    c.release_workspace()
    b = c.transform_host(rp, ci)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c.close()
    from paper_2007_11111_b200 import _core
    _core.release_device_memory()


def test_degenerate_shapes(ctx):
    """Shapes that leave parts of the pipeline empty: no active vertices
    (perfect matching, single edge), one vertex, isolated tail vertices, two
    disjoint triangles, a path, a 4-clique plus pendants, and a star with one
    hub whose N-(u) holds every other vertex."""
    m = 50
    matching = gu.from_pairs([(2 * i, 2 * i + 1) for i in range(m)], 2 * m)
    cases = [matching, gu.from_pairs([(0, 1)], 2), gu.from_pairs([], 1),
             gu.from_pairs([(0, 1), (1, 2), (2, 0)], 40),
             gu.from_pairs([(0, 1), (1, 2), (2, 0), (3, 4), (4, 5), (5, 3)], 6),
             gu.path(300), gu.complete(4),
             gu.from_pairs([(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4), (4, 5)], 6),
             gu.star(2000)]
    for rp, ci in cases:
        check_same(ctx, rp, ci)
        check_same(ctx, rp, ci, mask=_capi.dict_mask([12, 13, 15]))


def test_randomised_paths_fuzz():
    """Seeded random graphs under random combinations of the internal-path
    hooks (4-cycle class, root bin, hub rows, triangle list mode) against the
    oracle: interactions between paths, not just each path alone."""
    rng = np.random.default_rng(2026)
    c = _capi.Context(0)
    for it in range(120):
        kind = it % 4
        if kind == 0:
            rp, ci = graphs.rmat(int(rng.integers(8, 13)), int(rng.integers(4, 20)),
                                 seed=int(rng.integers(1, 1000)))
        elif kind == 1:
            rp, ci = gu.er(int(rng.integers(50, 400)), float(rng.uniform(0.02, 0.3)),
                           int(rng.integers(1, 1000)))
        elif kind == 2:
            rp, ci = graphs.sbm(int(rng.integers(8, 64)), int(rng.integers(8, 64)),
                                float(rng.uniform(0.1, 0.6)), float(rng.uniform(0.5, 4.0)),
                                int(rng.integers(1, 1000)))
        else:
            rp, ci = gu.regular(int(rng.integers(100, 600)), int(rng.integers(3, 30)),
                                int(rng.integers(1, 1000)))
        c.set_debug(_capi.DEBUG_C4_CLASS, int(rng.choice([0, 0, 2, 3, 4, 5])))
        c.set_debug(_capi.DEBUG_C4_PARTS, int(rng.choice([0, 1, 2, 5])))
        c.set_debug(_capi.DEBUG_ROOTS_BIN, int(rng.choice([0, 0, 1, 2, 3, 4, 5])))
        c.set_debug(_capi.DEBUG_HUB, int(rng.choice([0, 1, 2])))
        c.set_debug(_capi.DEBUG_TRILIST, int(rng.choice([0, 0, 1, 2])))
        mask = 0xFFFF if it % 3 else int(rng.integers(0, 1 << 16)) | 3
        check_same(c, rp, ci, mask=mask, lenient=True, d15_mode=1)
    c.close()
