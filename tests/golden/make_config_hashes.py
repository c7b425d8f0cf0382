"""Per-column SHA-256 golden hashes of the full-Σ16 raw and net tables of the
large BASELINE configs, computed OFFLINE on the CPU by the parity checker
(oracle/, test infrastructure) — the GPU path never runs here.

    python tests/golden/make_config_hashes.py 4        # R-MAT 23 (~15 min, 8 cores)
    python tests/golden/make_config_hashes.py 3 4 5

Method: ``oracle.binding.transform(..., d15_mode=2)`` — the C restatement of
the reference plan and column fill (oracle/fglt_oracle.c) with every W-cost
term (C3, c4/d14, d13, d15) from the degree-oriented restatements of
oracle/fglt_oriented.c. Those are pinned bit-exact to the UNMODIFIED
reference (oracle/_ref) by tests/test_oracle_pin.py::test_oriented_terms_pin
on R-MAT <= 14, SBM and RGG samples; the reference's own passes need ~1 h
(non-d15) plus ~700 core-hours (d15) at config 4, out of reach.

Output ``config<k>.json``: the generator string, n, nnz, CSR hashes (so the
GPU test proves it rebuilt the same instance), W, and sha256 of every raw and
net column (uint64 little-endian, row order = vertex id) plus column sums.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import binding as ob  # noqa: E402
from paper_2007_11111_b200 import graphs  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def column_record(raw, net):
    return {
        "raw_col_sha256": [sha(raw[:, j]) for j in range(raw.shape[1])],
        "net_col_sha256": [sha(net[:, j]) for j in range(net.shape[1])],
        "raw_colsums": [int(x) for x in raw.sum(0, dtype=np.uint64)],
        "net_colsums": [int(x) for x in net.sum(0, dtype=np.uint64)],
    }


def main(cfgs):
    for k in cfgs:
        name, rp, ci = graphs.config(k)
        t0 = time.time()
        raw, net = ob.transform(rp, ci, 0xFFFF, False, 2)
        dt = time.time() - t0
        W, dmax = ob.graph_stats(rp)
        rec = {"config": k, "generator": name, "n": len(rp) - 1, "nnz": len(ci),
               "row_ptr_sha256": sha(rp.astype(np.int32)),
               "col_idx_sha256": sha(ci.astype(np.int32)), "W": W, "d_max": dmax,
               "method": "oracle.binding.transform(d15_mode=2): C restatement + oriented W terms",
               "cpu_seconds": round(dt, 1), "oracle_threads": ob.num_threads()}
        rec.update(column_record(raw, net))
        with open(os.path.join(HERE, f"config{k}.json" if k != 1 else "config1_columns.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print(f"config {k}: n={rec['n']} nnz={rec['nnz']} {dt:.1f}s", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4])
