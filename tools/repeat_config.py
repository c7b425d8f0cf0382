"""Hash raw+net of repeated full transforms of a BASELINE config (determinism check; dev tool)."""
import sys, hashlib
sys.path.insert(0, ".")
import numpy as np
from paper_2007_11111_b200 import _capi, graphs
name, rp, ci = graphs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
c = _capi.Context(0)
hs = []
for r in range(3):
    raw, net, _ = c.transform_host(rp, ci)
    hs.append(hashlib.sha256(raw.tobytes() + net.tobytes()).hexdigest()[:16])
print(name, hs, "identical" if len(set(hs)) == 1 else "MISMATCH")
