"""Run the golden sub-dictionary fixtures through the C-ABI and print each
outcome (dev tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2007_11111_b200 import _capi  # noqa: E402

z = np.load("tests/golden/small_tables.npz")
ctx = _capi.Context(0)
rp, ci = z["rmat10_rp"], z["rmat10_ci"]
for key in sorted(z.files):
    if not key.startswith("rmat10_m") or key.endswith("_net"):
        continue
    mask, lenient = int(key[8:12], 16), bool(int(key[14]))
    try:
        raw, net, _ = ctx.transform_host(rp, ci, mask, lenient)
        if key.endswith("_err"):
            print(key, "GPU ok but reference raised", z[key].tolist())
        else:
            bad = raw != z[key]
            print(key, "raw ok" if not bad.any() else f"raw cols differ {np.nonzero(bad.any(0))[0].tolist()}",
                  "net ok" if (net == z[key[:-4] + '_net']).all() else "net differs")
    except _capi.TransformFailed as e:
        print(key, "GPU raised", (e.code, e.graphlet_id, e.vertex),
              "reference:", z[key].tolist() if key.endswith("_err") else "tables")
