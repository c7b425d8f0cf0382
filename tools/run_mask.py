"""Bisect helper: python tools/run_mask.py <rmat scale> <hex mask>"""
import sys

sys.path.insert(0, ".")
from paper_2007_11111_b200 import _capi, graphs  # noqa: E402

rp, ci = graphs.rmat(int(sys.argv[1]), 16, seed=1)
mask = int(sys.argv[2], 16)
ctx = _capi.Context(0)
raw, net, st = ctx.transform_host(rp, ci, mask, lenient=True)
print("ok", hex(mask))
