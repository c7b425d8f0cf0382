"""Regenerate the golden fixtures from the UNMODIFIED reference library
(oracle/_ref/libfglt_ref.so, built by oracle/Makefile from /root/reference).
Run in the dev container (the reference tree is not on the GPU box):

    python tests/golden/make_golden.py

Fixtures (all produced by the reference's own graphlet::transform):
  config1.json      er_graph(2000, 0.004, 1): CSR hash, raw/net sha256 + column sums
  small_tables.npz  full raw/net tables of small seeded graphs (R-MAT 10, SBM 16x64,
                    RGG 3000, K6, C8, star 7) and of sub-dictionary / lenient cases
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import binding as ob  # noqa: E402
from paper_2007_11111_b200 import graphs  # noqa: E402
import fglt_testutil as gu  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    rp, ci = ob.ref_er_graph(2000, 0.004, 1)
    raw, net, _, _ = ob.ref_transform(rp, ci, 0xFFFF, False, 1)
    cfg1 = {"generator": "testutil::er_graph(2000, 0.004, 1) (proj/tests/testutil.hpp:90-99)",
            "n": len(rp) - 1, "nnz": len(ci), "col_idx_sha256": sha(ci.astype(np.int32)),
            "row_ptr_sha256": sha(rp.astype(np.int32)),
            "raw_sha256": sha(raw), "net_sha256": sha(net),
            "raw_colsums": [int(x) for x in raw.sum(0)], "net_colsums": [int(x) for x in net.sum(0)]}
    with open(os.path.join(HERE, "config1.json"), "w") as f:
        json.dump(cfg1, f, indent=1)

    cases = {
        "rmat10": graphs.rmat(10, 16, seed=10),
        "sbm16": graphs.sbm(16, 64, 0.3, 3.0, 16),
        "rgg3000": graphs.rgg(3000, 6.0, 30),
        "k6": gu.complete(6),
        "c8": gu.cycle(8),
        "star7": gu.star(7),
        "demo": gu.demo(),
    }
    out = {}
    for name, (rp, ci) in cases.items():
        raw, net, _, _ = ob.ref_transform(rp, ci, 0xFFFF, False, 1)
        out[f"{name}_rp"], out[f"{name}_ci"] = rp.astype(np.int32), ci.astype(np.int32)
        out[f"{name}_raw"], out[f"{name}_net"] = raw, net
    # sub-dictionaries on rmat10, strict and lenient, incl. an error case
    rp, ci = cases["rmat10"]
    for mask in (0x001F, 0x1003, 0x8013, 0x2023, 0x7FFF):
        for lenient in (0, 1):
            key = f"rmat10_m{mask:04x}_l{lenient}"
            try:
                raw, net, _, _ = ob.ref_transform(rp, ci, mask, bool(lenient), 1)
                out[key + "_raw"], out[key + "_net"] = raw, net
            except ob.OracleError as e:
                out[key + "_err"] = np.array([e.code, e.graphlet_id, e.vertex], np.int64)
    np.savez_compressed(os.path.join(HERE, "small_tables.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
