"""Generate tests/golden/config4.json: the oracle's full Σ16 raw + net tables
for BASELINE.json config 4 (R-MAT scale 23, ~129M edges), summarised as
SHA-256 digests and column sums so the GPU test can compare at full size
without re-running a ~1 h CPU oracle on the box.

The oracle is the C restatement (oracle/fglt_oracle.c), d15 by its oriented
K4 counter (pinned bit-exact to the reference's compute_d15 on configs 1, 2, 5
and R-MAT <= 16, tests/test_oracle_pin.py). The graph is the committed
generator's, so the GPU side rebuilds the identical CSR (its SHA-256 is
recorded too).

  OMP_NUM_THREADS=8 python tests/golden/make_config4_golden.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import binding as ob  # noqa: E402
from paper_2007_11111_b200 import graphs  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8)).hexdigest()


def main(cfg: int = 4):
    t0 = time.time()
    name, rp, ci = graphs.config(cfg)
    print(name, "n", len(rp) - 1, "nnz", len(ci), "gen", round(time.time() - t0, 1), "s",
          flush=True)
    t1 = time.time()
    raw, net = ob.transform(rp, ci, 0xFFFF, False, 0)
    secs = time.time() - t1
    print("oracle", round(secs, 1), "s", flush=True)
    out = {
        "config": cfg, "name": name, "n": len(rp) - 1, "nnz": len(ci),
        "row_ptr_sha256": sha(rp.astype(np.int32)), "col_idx_sha256": sha(ci.astype(np.int32)),
        "raw_sha256": sha(raw), "net_sha256": sha(net),
        "raw_colsums": [str(int(x)) for x in raw.sum(axis=0, dtype=np.uint64)],
        "net_colsums": [str(int(x)) for x in net.sum(axis=0, dtype=np.uint64)],
        "oracle": "oracle/fglt_oracle.c fglt_oracle_transform, d15 oriented K4 counter",
        "oracle_seconds": round(secs, 1), "oracle_threads": ob.num_threads(),
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"config{cfg}.json")
    if cfg != 4:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"config{cfg}_full.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
