"""Find the first acceptance-family graph where GPU != oracle (dev tool)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import fglt_testutil as gu  # noqa: E402
from oracle import binding as ob  # noqa: E402
from paper_2007_11111_b200 import _capi  # noqa: E402

seed = 0x51AB5EED
cases = []
for i in range(120):
    n = 5 + (i * 7) % 36
    p = 0.1 if i % 3 == 0 else 0.2 if i % 3 == 1 else 0.4
    cases.append(("er%d" % i, gu.er(n, p, seed + i)))
for d in (3, 4, 5):
    for j in range(20):
        cases.append(("reg%d_%d" % (d, j), gu.regular(6 + 2 * (j % 18), d, seed + 1000 + j + d)))
for n in (2, 5, 9, 14, 20, 27, 33, 40, 15, 25):
    cases.append(("tree%d" % n, gu.tree(n, seed + 31 * n)))
cases += [("K%d" % n, gu.complete(n)) for n in range(2, 7)]
cases += [("C%d" % n, gu.cycle(n)) for n in range(3, 9)]
cases += [("star%d" % k, gu.star(k)) for k in range(2, 9)]
ctx = _capi.Context(0)
nbad = 0
for name, (rp, ci) in cases:
    oraw, onet = ob.transform(rp, ci)
    try:
        raw, net, _ = ctx.transform_host(rp, ci)
        ok = np.array_equal(raw, oraw) and np.array_equal(net, onet)
        err = None
    except _capi.TransformFailed as e:
        ok, err = False, str(e)
    if not ok:
        nbad += 1
        if nbad <= 3:
            d = np.diff(rp)
            print(name, "n", len(rp) - 1, "m", len(ci) // 2, "deg<=1:", int((d <= 1).sum()), err)
            if err is None:
                bad = raw != oraw
                print("  cols", np.nonzero(bad.any(0))[0].tolist(), "rows", np.nonzero(bad.any(1))[0][:8].tolist())
print("bad", nbad, "of", len(cases))
