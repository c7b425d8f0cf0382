"""Repeat a transform R times on one graph; compare each run with the oracle
and report differing columns (dev tool for nondeterminism hunts)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import binding as ob  # noqa: E402
from paper_2007_11111_b200 import _capi, graphs  # noqa: E402

scale, reps = int(sys.argv[1]), int(sys.argv[2])
rp, ci = graphs.rmat(scale, 16, seed=1)
oraw, onet = ob.transform(rp, ci, 0xFFFF, False, 1)
ctx = _capi.Context(0)
for r in range(reps):
    raw, net, st = ctx.transform_host(rp, ci)
    bad = raw != oraw
    if bad.any():
        cols = np.nonzero(bad.any(0))[0]
        print(f"run {r}: MISMATCH cols {cols.tolist()} rows {int(bad.any(1).sum())}", flush=True)
        for c in cols[:3]:
            rr = np.nonzero(bad[:, c])[0][:4]
            print("   col", c, "rows", rr.tolist(), "gpu", raw[rr, c].tolist(), "oracle",
                  oraw[rr, c].tolist(), flush=True)
    else:
        print(f"run {r}: ok", flush=True)
