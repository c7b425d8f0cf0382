"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the parity checkers.

* ``liboracle.so``: the C restatement (oracle/fglt_oracle.c)
* ``_ref/libfglt_ref.so``: the unmodified reference library (oracle/Makefile)

Imported only by tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs — never by the product package.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfglt_ref.so")

vp = ctypes.c_void_p
i64 = ctypes.c_int64

_o = None
_r = None


def oracle():
    global _o
    if _o is None:
        L = ctypes.CDLL(ORACLE_SO)
        L.fglt_oracle_transform.restype = ctypes.c_int
        L.fglt_oracle_transform.argtypes = [vp, vp, i64, ctypes.c_uint32, ctypes.c_int,
                                            ctypes.c_int, vp, vp, vp, vp, vp]
        for name in ("fglt_oracle_p1",):
            getattr(L, name).argtypes = [vp, i64, vp]
        L.fglt_oracle_p2.argtypes = [vp, vp, i64, vp, vp]
        L.fglt_oracle_c3.argtypes = [vp, vp, i64, vp, vp]
        L.fglt_oracle_p3.argtypes = [vp, vp, i64, vp, vp, vp, vp]
        L.fglt_oracle_c4_d14.restype = ctypes.c_uint64
        L.fglt_oracle_c4_d14.argtypes = [vp, vp, i64, vp, vp]
        L.fglt_oracle_d13.argtypes = [vp, vp, i64, vp, vp]
        L.fglt_oracle_d15_ref_algorithm.argtypes = [vp, vp, i64, vp]
        L.fglt_oracle_d15_oriented.argtypes = [vp, vp, i64, vp]
        L.fglt_oracle_u16.argtypes = [vp]
        L.fglt_oracle_net_from_raw.argtypes = [vp, vp, i64, ctypes.c_uint32, ctypes.c_int, vp, vp, vp]
        L.fglt_oracle_graph_stats.argtypes = [vp, i64, vp, vp]
        L.fglt_oracle_num_threads.restype = ctypes.c_int
        _o = L
    return _o


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _r
    if _r is None:
        L = ctypes.CDLL(REF_SO)
        L.fglt_ref_transform_csr32.restype = ctypes.c_int
        L.fglt_ref_transform_csr32.argtypes = [vp, vp, i64, i64, ctypes.c_uint32, ctypes.c_int,
                                               ctypes.c_int, vp, vp, vp, vp, vp, ctypes.c_char_p,
                                               ctypes.c_int]
        L.fglt_ref_last_stats.restype = ctypes.c_char_p
        L.fglt_ref_er_graph.restype = i64
        L.fglt_ref_er_graph.argtypes = [i64, ctypes.c_double, ctypes.c_uint64, vp, vp]
        L.fglt_ref_oracle.restype = ctypes.c_int
        L.fglt_ref_oracle.argtypes = [vp, vp, i64, i64, vp, vp]
        L.fglt_ref_counts.argtypes = [vp, vp, i64, i64, vp]
        L.fglt_ref_build_adjacency.restype = ctypes.c_int
        L.fglt_ref_build_adjacency.argtypes = [vp, vp, i64, i64, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, vp, vp, vp, ctypes.c_char_p,
                                               ctypes.c_int]
        L.fglt_ref_d15.restype = ctypes.c_int
        L.fglt_ref_d15.argtypes = [vp, vp, i64, i64, ctypes.c_int, vp]
        _r = L
    return _r


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ids(mask):
    mask |= 3
    return [i for i in range(16) if mask >> i & 1]


class OracleError(Exception):
    def __init__(self, code, graphlet, vertex):
        super().__init__(f"code={code} graphlet={graphlet} vertex={vertex}")
        self.code, self.graphlet_id, self.vertex = code, graphlet, vertex


def transform(rp, ci, mask=0xFFFF, lenient=False, d15_mode=0):
    """Oracle raw + net (n x k) following the reference plan; raises
    OracleError(code, graphlet, vertex) like the reference's exceptions."""
    rp, ci = _c(rp, np.int32), _c(ci, np.int32)
    n = len(rp) - 1
    k = len(_ids(mask))
    raw = np.zeros((n, k), np.uint64)
    net = np.zeros((n, k), np.uint64)
    g = np.zeros(1, np.int32)
    v = np.zeros(1, np.int64)
    t = np.zeros(1, np.uint64)
    rc = oracle().fglt_oracle_transform(rp.ctypes.data, ci.ctypes.data, n, mask, int(lenient),
                                        d15_mode, raw.ctypes.data, net.ctypes.data, g.ctypes.data,
                                        v.ctypes.data, t.ctypes.data)
    if rc:
        raise OracleError(rc, int(g[0]), int(v[0]))
    return raw, net


def vectors(rp, ci):
    """Per-kernel reference quantities (p1, p2, c3, C3, p3, c4, d14, d13)."""
    rp, ci = _c(rp, np.int32), _c(ci, np.int32)
    n, nnz = len(rp) - 1, len(ci)
    L = oracle()
    out = {k: np.zeros(n, np.uint64) for k in ("p1", "p2", "c3", "p3", "c4", "d14", "d13")}
    C3 = np.zeros(max(nnz, 1), np.uint64)
    L.fglt_oracle_p1(rp.ctypes.data, n, out["p1"].ctypes.data)
    L.fglt_oracle_p2(rp.ctypes.data, ci.ctypes.data, n, out["p1"].ctypes.data, out["p2"].ctypes.data)
    L.fglt_oracle_c3(rp.ctypes.data, ci.ctypes.data, n, out["c3"].ctypes.data, C3.ctypes.data)
    L.fglt_oracle_p3(rp.ctypes.data, ci.ctypes.data, n, out["p1"].ctypes.data, out["p2"].ctypes.data,
                     out["c3"].ctypes.data, out["p3"].ctypes.data)
    touches = L.fglt_oracle_c4_d14(rp.ctypes.data, ci.ctypes.data, n, out["c4"].ctypes.data,
                                   out["d14"].ctypes.data)
    L.fglt_oracle_d13(rp.ctypes.data, ci.ctypes.data, n, C3.ctypes.data, out["d13"].ctypes.data)
    out["C3"] = C3[:nnz]
    out["touches"] = int(touches)
    return out


def d15(rp, ci, mode="oriented"):
    rp, ci = _c(rp, np.int32), _c(ci, np.int32)
    n = len(rp) - 1
    out = np.zeros(n, np.uint64)
    fn = oracle().fglt_oracle_d15_oriented if mode == "oriented" else \
        oracle().fglt_oracle_d15_ref_algorithm
    fn(rp.ctypes.data, ci.ctypes.data, n, out.ctypes.data)
    return out


def u16():
    out = np.zeros(256, np.uint64)
    oracle().fglt_oracle_u16(out.ctypes.data)
    return out.reshape(16, 16)


def net_from_raw(raw, mask, lenient=False):
    raw = _c(raw, np.uint64)
    net = np.zeros_like(raw)
    g = np.zeros(1, np.int32)
    v = np.zeros(1, np.int64)
    code = np.zeros(1, np.int32)
    oracle().fglt_oracle_net_from_raw(raw.ctypes.data, net.ctypes.data, raw.shape[0], mask,
                                      int(lenient), g.ctypes.data, v.ctypes.data, code.ctypes.data)
    if code[0]:
        raise OracleError(int(code[0]), int(g[0]), int(v[0]))
    return net


def graph_stats(rp):
    rp = _c(rp, np.int32)
    W = np.zeros(1, np.uint64)
    dm = np.zeros(1, np.uint64)
    oracle().fglt_oracle_graph_stats(rp.ctypes.data, len(rp) - 1, W.ctypes.data, dm.ctypes.data)
    return int(W[0]), int(dm[0])


def num_threads():
    return oracle().fglt_oracle_num_threads()


# ----------------------------------------------------------- the reference
def ref_transform(rp, ci, mask=0xFFFF, lenient=False, threads=0):
    """The unmodified reference graphlet::transform on the same CSR.
    Returns (raw, net, seconds, stats) or raises OracleError."""
    rp, ci = _c(rp, np.int32), _c(ci, np.int32)
    n, nnz = len(rp) - 1, len(ci)
    k = len(_ids(mask))
    raw = np.zeros((n, k), np.uint64)
    net = np.zeros((n, k), np.uint64)
    secs = np.zeros(1, np.float64)
    g = np.zeros(1, np.int32)
    v = np.zeros(1, np.int64)
    msg = ctypes.create_string_buffer(256)
    rc = ref().fglt_ref_transform_csr32(rp.ctypes.data, ci.ctypes.data, n, nnz, mask,
                                        int(lenient), threads, raw.ctypes.data, net.ctypes.data,
                                        secs.ctypes.data, g.ctypes.data, v.ctypes.data, msg, 256)
    if rc:
        raise OracleError(rc, int(g[0]), int(v[0]))
    return raw, net, float(secs[0]), json.loads(ref().fglt_ref_last_stats().decode())


def ref_er_graph(n, p, seed):
    L = ref()
    nnz = L.fglt_ref_er_graph(n, p, seed, None, None)
    rp = np.zeros(n + 1, np.int32)
    ci = np.zeros(nnz, np.int32)
    L.fglt_ref_er_graph(n, p, seed, rp.ctypes.data, ci.ctypes.data)
    return rp, ci


def ref_oracle(rp, ci):
    rp, ci = _c(rp, np.int32), _c(ci, np.int32)
    n = len(rp) - 1
    raw = np.zeros((n, 16), np.uint64)
    net = np.zeros((n, 16), np.uint64)
    rc = ref().fglt_ref_oracle(rp.ctypes.data, ci.ctypes.data, n, len(ci), raw.ctypes.data,
                               net.ctypes.data)
    if rc:
        raise OracleError(rc, -1, -1)
    return raw, net


def ref_counts(rp, ci):
    rp, ci = _c(rp, np.int32), _c(ci, np.int32)
    out = np.zeros(3, np.uint64)
    ref().fglt_ref_counts(rp.ctypes.data, ci.ctypes.data, len(rp) - 1, len(ci), out.ctypes.data)
    return [int(x) for x in out]


def ref_d15(rp, ci, threads=0):
    rp, ci = _c(rp, np.int32), _c(ci, np.int32)
    out = np.zeros(len(rp) - 1, np.uint64)
    ref().fglt_ref_d15(rp.ctypes.data, ci.ctypes.data, len(rp) - 1, len(ci), threads,
                       out.ctypes.data)
    return out


def ref_build_adjacency(eu, ev, declared_n=0, symmetrize=True, drop_self_loops=True, dedupe=True):
    """The reference's build_adjacency on int64 pairs. Returns (rp, ci,
    self_loops_dropped, duplicates_merged) or raises OracleError(2, msg)."""
    eu, ev = _c(eu, np.int64), _c(ev, np.int64)
    ne = len(eu)
    nmax = max(int(declared_n), int(max(eu.max(initial=-1), ev.max(initial=-1))) + 1, 0)
    rp = np.zeros(nmax + 1, np.int32)
    ci = np.zeros(max(2 * ne, 1), np.int32)
    out = np.zeros(4, np.int64)
    msg = ctypes.create_string_buffer(256)
    rc = ref().fglt_ref_build_adjacency(eu.ctypes.data, ev.ctypes.data, ne, int(declared_n),
                                        int(symmetrize), int(drop_self_loops), int(dedupe),
                                        rp.ctypes.data, ci.ctypes.data, out.ctypes.data, msg, 256)
    if rc:
        e = OracleError(rc, -1, -1)
        e.msg = msg.value.decode()
        raise e
    n, nnz = int(out[0]), int(out[1])
    return rp[:n + 1].copy(), ci[:nnz].copy(), int(out[2]), int(out[3])


def ref_parse_dictionary(spec: str):
    """The reference's parse_dictionary: (ids, implicitly_added) or raises
    ValueError(message)."""
    L = ref()
    L.fglt_ref_parse_dictionary.restype = ctypes.c_int
    L.fglt_ref_parse_dictionary.argtypes = [ctypes.c_char_p, vp, vp, ctypes.c_char_p, ctypes.c_int]
    ids = np.zeros(1, np.uint32)
    imp = np.zeros(1, np.uint32)
    msg = ctypes.create_string_buffer(256)
    if L.fglt_ref_parse_dictionary(spec.encode(), ids.ctypes.data, imp.ctypes.data, msg, 256):
        raise ValueError(msg.value.decode())
    return ([i for i in range(16) if int(ids[0]) >> i & 1],
            [i for i in range(16) if int(imp[0]) >> i & 1])
