"""Run the transform R times per setting and compare runs against the first
run (dev tool for nondeterminism hunts). Prints per-setting mismatch counts."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2007_11111_b200 import _capi, graphs  # noqa: E402

scale, reps = int(sys.argv[1]), int(sys.argv[2])
rp, ci = graphs.rmat(scale, 16, seed=1)
settings = [("default", {}, 0xFFFF), ("roots->bin4", {3: 4}, 0xFFFF),
            ("roots->slab", {3: 5}, 0xFFFF), ("d13 only", {}, (1 << 13) | 3),
            ("c4->hash", {1: 2}, 0xFFFF), ("c4->tiles32", {1: 4}, 0xFFFF)]
pick = sys.argv[3].split(",") if len(sys.argv) > 3 else None
for name, dbg, mask in settings:
    if pick and name not in pick:
        continue
    ctx = _capi.Context(0)
    for k, v in dbg.items():
        ctx.set_debug(k, v)
    base = None
    bad = 0
    details = []
    for r in range(reps):
        raw, _, _ = ctx.transform_host(rp, ci, mask, lenient=True)
        if base is None:
            base = raw.copy()
            continue
        d = raw != base
        if d.any():
            bad += 1
            cols = np.nonzero(d.any(0))[0].tolist()
            rows = np.nonzero(d.any(1))[0][:3].tolist()
            details.append((r, cols, rows, [int(raw[x, cols[0]]) - int(base[x, cols[0]]) for x in rows]))
    print(f"{name:14s} mismatching runs {bad}/{reps - 1}", details[:4], flush=True)
    ctx.close()
