"""Per-buffer device scratch of one transform (dev tool, needs a GPU): the
criterion-6 graphs of the reference acceptance harness (random 4-regular-like
graphs, n = 10^4 .. 8*10^4) and any BASELINE config.
  python tools/scratch_report.py            # small graphs
  python tools/scratch_report.py 3          # config 3
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2007_11111_b200 import _capi, graphs  # noqa: E402


def regular_like(n, d, seed):
    rng = np.random.default_rng(seed)
    u = np.repeat(np.arange(n), d // 2)
    v = (u + rng.integers(1, n, len(u))) % n
    rp, ci, _ = graphs.csr_from_pairs(u, v, n)
    return rp, ci


ctx = _capi.Context(0)
cases = [(f"config {a}", *graphs.config(int(a))[1:]) for a in sys.argv[1:]] or \
        [(f"regular-like n={n}", *regular_like(n, 4, n)) for n in (10000, 20000, 40000, 80000)]
for name, rp, ci in cases:
    n, m = len(rp) - 1, len(ci) // 2
    raw, net, st = ctx.transform_host(rp, ci, 0xFFFF)
    rep = ctx.scratch_report()
    bound = 3 * m + 12 * n + 64
    print(f"{name}: n={n} m={m} peak_aux_words={st['peak_aux_words']} bound(3m+12n+64)={bound} "
          f"ratio={st['peak_aux_words'] / bound:.2f} largest={st['largest_aux_alloc_words']}")
    for b, (bytes_, staging) in sorted(rep.items(), key=lambda kv: -kv[1][0]):
        print(f"   {b:10s} {bytes_ / 8:14.0f} words {bytes_ / 8 / n:8.2f}/n {'(staging)' if staging else ''}")
