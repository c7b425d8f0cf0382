"""The compute-sanitizer workload (VERDICT r1 "next" #7): small transforms
that reach every device code path — config 1, config 2's generator at 20 000
points, R-MAT 12 under each forced internal path (4-cycle classes, root bins,
hub rows, triangle list on / off / exhausted), a sub-dictionary and the
staged (sharded) API — each checked against the oracle. Run as
  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_cases.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import binding as ob  # noqa: E402
from paper_2007_11111_b200 import _capi, graphs  # noqa: E402

FORCED = [  # (debug key, value, parts)
    (None, None, None),
    (_capi.DEBUG_C4_CLASS, 2, 1), (_capi.DEBUG_C4_CLASS, 2, 3), (_capi.DEBUG_C4_CLASS, 3, None),
    (_capi.DEBUG_C4_CLASS, 4, None), (_capi.DEBUG_C4_CLASS, 5, None),
    (_capi.DEBUG_ROOTS_BIN, 1, None), (_capi.DEBUG_ROOTS_BIN, 4, None),
    (_capi.DEBUG_ROOTS_BIN, 5, None),
    (_capi.DEBUG_HUB, 1, None), (_capi.DEBUG_HUB, 2, None),
    (_capi.DEBUG_TRILIST, 1, None), (_capi.DEBUG_TRILIST, 2, None),
]


def check(ctx, rp, ci, mask=0xFFFF, label=""):
    raw, net, _ = ctx.transform_host(rp, ci, mask)
    oraw, onet = ob.transform(rp, ci, mask, False, 1)
    ok = np.array_equal(raw, oraw) and np.array_equal(net, onet)
    print(f"{label}: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    ok = True
    ctx = _capi.Context(0)
    ok &= check(ctx, *graphs.config(1)[1:], label="config 1")
    ok &= check(ctx, *graphs.rgg(20000, 3.0, 2), label="rgg 20000")
    ok &= check(ctx, *graphs.sbm(64, 64, 0.3, 3.0, 5), label="sbm 64x64")
    rp, ci = graphs.rmat(12, 16, seed=1)
    for key, val, parts in FORCED:
        c = _capi.Context(0)
        if key is not None:
            c.set_debug(key, val)
        if parts is not None:
            c.set_debug(_capi.DEBUG_C4_PARTS, parts)
        ok &= check(c, rp, ci, label=f"rmat12 forced {key}={val} parts={parts}")
        c.close()
    ok &= check(ctx, rp, ci, mask=0x801F, label="rmat12 dict {0-4,15}")
    raw, net, _ = _capi.transform_multi(rp, ci, [0, 0])
    oraw, onet = ob.transform(rp, ci, 0xFFFF, False, 1)
    ok &= np.array_equal(raw, oraw) and np.array_equal(net, onet)
    print("staged x2:", "ok" if ok else "MISMATCH")
    ctx.close()
    print("ALL OK" if ok else "SOME MISMATCH")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
