"""Run one transform on a generated graph and check it against the oracle
(dev tool for bisecting failures):
  python tools/run_case.py rmat 17 [check] [debugkey=value ...]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2007_11111_b200 import _capi, graphs  # noqa: E402

kind, arg = sys.argv[1], int(sys.argv[2])
check = len(sys.argv) > 3 and sys.argv[3] == "check"
if kind == "rmat":
    rp, ci = graphs.rmat(arg, 16, seed=1)
elif kind == "sbm":
    rp, ci = graphs.sbm(arg, 64, 0.3, 3.0, 5)
else:
    rp, ci = graphs.config(arg)[1:]
ctx = _capi.Context(0)
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    ctx.set_debug(int(k), int(v))
raw, net, st = ctx.transform_host(rp, ci)
print(kind, arg, "ok", st["kernel_launches"], sys.argv[4:], flush=True)
if check:
    from oracle import binding as ob
    oraw, onet = ob.transform(rp, ci, 0xFFFF, False, 1)
    print("parity", np.array_equal(raw, oraw), np.array_equal(net, onet))
    bad = raw != oraw
    if bad.any():
        cols = np.nonzero(bad.any(0))[0]
        print("raw columns differing:", cols.tolist(), "rows:", int(bad.any(1).sum()))
        for c in cols[:4]:
            r = np.nonzero(bad[:, c])[0][:5]
            print("  col", c, "rows", r.tolist(), "gpu", raw[r, c].tolist(), "oracle", oraw[r, c].tolist())
