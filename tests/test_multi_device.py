"""Single-process multi-device transform (fglt_transform_multi, SURVEY §8b
devices[] + §8e sharding): byte-identical to the one-device transform for any
device list. On a one-GPU machine, repeated device ids run the same ranks in
sequence with host-staged sums (tests the rank decomposition and the error
combination); a real NCCL clique runs when >= 2 GPUs are present."""
import numpy as np
import pytest

from paper_2007_11111_b200 import _capi, graphs
import fglt_testutil as gu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = _capi.Context(0)
    yield c
    c.close()


CASES = {
    "demo": gu.demo(),
    "rmat12": graphs.rmat(12, 16, seed=5),
    "sbm": graphs.sbm(128, 64, 0.3, 3.0, 8),
    "rgg": graphs.rgg(20000, 3.0, 9),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_equals_single(ctx, name, devices):
    rp, ci = CASES[name]
    raw1, net1, _ = ctx.transform_host(rp, ci, 0xFFFF)
    raw, net, st = _capi.transform_multi(rp, ci, devices)
    assert np.array_equal(raw, raw1) and np.array_equal(net, net1)
    assert st["kernel_launches"] > 0


def test_multi_sub_dictionary_and_errors(ctx):
    rp, ci = CASES["rmat12"]
    for mask in (0x1003, 0x801F, 0x7FFF):
        try:
            raw1, net1, _ = ctx.transform_host(rp, ci, mask)
        except _capi.TransformFailed as e:
            with pytest.raises(_capi.TransformFailed) as e2:
                _capi.transform_multi(rp, ci, [0, 0], mask)
            assert (e2.value.code, e2.value.graphlet_id, e2.value.vertex) == \
                (e.code, e.graphlet_id, e.vertex)
            continue
        raw, net, _ = _capi.transform_multi(rp, ci, [0, 0], mask)
        assert np.array_equal(raw, raw1) and np.array_equal(net, net1)


def test_multi_rejects_bad_devices():
    rp, ci = gu.demo()
    with pytest.raises(_capi.TransformFailed) as e:
        _capi.transform_multi(rp, ci, [0, 99])
    assert e.value.code == 7


def test_multi_nccl_clique_when_available(ctx):
    n = _capi.lib().fglt_device_count()
    if n < 2:
        pytest.skip("one GPU: the NCCL clique path needs >= 2 devices")
    rp, ci = CASES["rmat12"]
    raw1, net1, _ = ctx.transform_host(rp, ci, 0xFFFF)
    raw, net, _ = _capi.transform_multi(rp, ci, list(range(n)))
    assert np.array_equal(raw, raw1) and np.array_equal(net, net1)


def test_python_and_cli_devices_option(tmp_path):
    """graphlet::transform with TransformOptions::devices (the Python
    `devices=` keyword and `glt --devices`) routes to fglt_transform_multi."""
    import os
    import subprocess

    import paper_2007_11111_b200 as gt
    rp, ci = CASES["sbm"]
    g = gt.from_csr(rp, ci)
    raw1, net1 = gt.transform(g)
    raw2, net2 = gt.transform(g, devices=[0, 0])
    assert np.array_equal(raw1, raw2) and np.array_equal(net1, net2)
    edges = tmp_path / "g.edges"
    with open(edges, "w") as f:
        for u in range(len(rp) - 1):
            for v in ci[rp[u]:rp[u + 1]]:
                if v > u:
                    f.write(f"{u} {v}\n")
    glt = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2007_11111_b200", "glt")
    outs = []
    for extra in ([], ["--devices", "0,0,0"]):
        out = tmp_path / ("o" + str(len(extra)))
        subprocess.run([glt, str(edges), "--emit", "both", "-o", str(out), *extra], check=True)
        outs.append(open(str(out) + ".raw").read() + open(str(out) + ".net").read())
    assert outs[0] == outs[1]
