"""Multi-rank orchestration (paper_2007_11111_b200/dist.py) under gloo on
CPU, world sizes 1, 2 and 3: CSR broadcast, root partition, the two integer
all-reduces, row-block epilogue, gather to rank 0, and rank-combined error
reporting. Device work is replaced by the independent numpy stand-in
(tests/numpy_stages.py); the result must equal the oracle byte for byte."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, mask, lenient, outq):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from numpy_stages import NumpyStages

    from paper_2007_11111_b200 import _capi
    from paper_2007_11111_b200.dist import sharded_transform
    rp, ci = case
    n, nnz = len(rp) - 1, len(ci)
    if rank == 0:
        rp_t, ci_t = torch.from_numpy(rp.astype(np.int32)), torch.from_numpy(ci.astype(np.int32))
    else:  # only the root holds the input; others receive it by broadcast
        rp_t, ci_t = torch.zeros(n + 1, dtype=torch.int32), torch.zeros(nnz, dtype=torch.int32)
    try:
        raw, net = sharded_transform(NumpyStages(), rp_t, ci_t, n, nnz, mask, lenient)
        if rank == 0:
            outq.put(("ok", raw.numpy().view(np.uint64).copy(), net.numpy().view(np.uint64).copy()))
    except _capi.TransformFailed as e:
        if rank == 0:
            outq.put(("err", e.code, e.graphlet_id, e.vertex))
    dist.destroy_process_group()


def run_world(world, case, mask=0xFFFF, lenient=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, mask, lenient, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def cases():
    import fglt_testutil as gu
    from paper_2007_11111_b200 import graphs
    return {"demo": gu.demo(), "er40": gu.er(40, 0.25, 7), "rmat7": graphs.rmat(7, 8, seed=3),
            "k6": gu.complete(6)}


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_equals_oracle(world):
    from oracle import binding as ob
    for name, case in cases().items():
        res = run_world(world, case)
        assert res[0] == "ok", (name, res)
        oraw, onet = ob.transform(*case)
        np.testing.assert_array_equal(res[1], oraw, err_msg=name)
        np.testing.assert_array_equal(res[2], onet, err_msg=name)


def test_sharded_error_is_lowest_vertex():
    """Incomplete family on K4: every vertex fails; ranks combine to the
    reference's choice (lowest vertex of the first failing stage)."""
    import fglt_testutil as gu
    from oracle import binding as ob
    case = gu.complete(4)
    mask = (1 << 5) | (1 << 13) | 3
    res = run_world(2, case, mask)
    with pytest.raises(ob.OracleError) as ei:
        ob.transform(*case, mask)
    assert res[0] == "err"
    assert (res[1], res[2], res[3]) == (ei.value.code, ei.value.graphlet_id, ei.value.vertex)
