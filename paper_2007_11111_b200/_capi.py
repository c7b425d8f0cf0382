"""ctypes view of the C-ABI (include/fglt.h) exported by the in-tree
``libfglt.so`` (sm_100a). This is the boundary the parity tests and the bench
call; there is no CPU fallback — loading fails loudly when the library or a
CUDA device is missing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FGLT_LIB_OVERRIDE") or os.path.join(_HERE, "libfglt.so")

FGLT_INPUT_DEVICE = 0x1
FGLT_OUTPUT_DEVICE = 0x2
FGLT_TIMINGS = 0x4

CODES = {0: "ok", 1: "parse", 2: "structural", 3: "overflow", 4: "inconsistency",
         5: "io", 6: "cuda", 7: "no-device"}

EXPORTS = [
    "fglt_ctx_create", "fglt_ctx_destroy", "fglt_ctx_release_workspace", "fglt_ctx_transform", "fglt_transform_csr32",
    "fglt_net_from_raw", "fglt_net_from_raw_matrix", "fglt_stage_prepare", "fglt_stage_bounds", "fglt_stage_triangles",
    "fglt_stage_local", "fglt_stage_local_part", "fglt_stage_roots", "fglt_stage_epilogue", "fglt_version",
    "fglt_device_count", "fglt_ctx_kernel_launches", "fglt_ctx_set_debug", "fglt_build_csr",
    "fglt_csr_fetch", "fglt_kernel_p2", "fglt_kernel_c3", "fglt_kernel_p3", "fglt_kernel_d7",
    "fglt_kernel_d8", "fglt_kernel_d9_d10_d11", "fglt_kernel_d13", "fglt_probe_smem_atomics",
    "fglt_ctx_scratch_report", "fglt_transform_multi",
]

DEBUG_C4_CLASS, DEBUG_C4_PARTS, DEBUG_ROOTS_BIN, DEBUG_HUB, DEBUG_TRILIST, DEBUG_ROW_SORT = 1, 2, 3, 4, 5, 6
DEBUG_FLAT_DMAX = 7


class FgltError(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("graphlet_id", ctypes.c_int32),
                ("vertex", ctypes.c_int64), ("msg", ctypes.c_char * 256),
                ("order_key", ctypes.c_uint64)]


MAX_STEPS = 12
MAX_PHASES = 16


class FgltStats(ctypes.Structure):
    _fields_ = [("num_steps", ctypes.c_int32),
                ("step_names", (ctypes.c_char * 32) * MAX_STEPS),
                ("step_seconds", ctypes.c_double * MAX_STEPS),
                ("p2_row_touches", ctypes.c_uint64), ("p2_touch_bound", ctypes.c_uint64),
                ("peak_aux_words", ctypes.c_uint64), ("largest_aux_alloc_words", ctypes.c_uint64),
                ("threads_used", ctypes.c_int32), ("device", ctypes.c_int32),
                ("W", ctypes.c_uint64), ("d_max", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64),
                ("num_phases", ctypes.c_int32),
                ("phase_names", (ctypes.c_char * 32) * MAX_PHASES),
                ("phase_seconds", ctypes.c_double * MAX_PHASES),
                ("phase_units", ctypes.c_uint64 * MAX_PHASES)]

    def as_dict(self):
        return {
            "kernel_times": [(self.step_names[i].value.decode(), self.step_seconds[i])
                             for i in range(self.num_steps)],
            "p2_row_touches": self.p2_row_touches, "p2_touch_bound": self.p2_touch_bound,
            "peak_aux_words": self.peak_aux_words,
            "largest_aux_alloc_words": self.largest_aux_alloc_words,
            "threads_used": self.threads_used, "device": self.device, "W": self.W,
            "d_max": self.d_max, "kernel_launches": self.kernel_launches,
            "phases": [(self.phase_names[i].value.decode(), self.phase_seconds[i],
                        int(self.phase_units[i])) for i in range(self.num_phases)],
        }


_lib = None


def lib():
    """Load libfglt.so (raises if absent: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32p, u64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p
        L.fglt_ctx_create.restype = vp
        L.fglt_ctx_create.argtypes = [ctypes.c_int, vp, ctypes.POINTER(FgltError)]
        L.fglt_ctx_destroy.restype = None
        L.fglt_ctx_destroy.argtypes = [vp]
        L.fglt_ctx_release_workspace.restype = ctypes.c_int
        L.fglt_ctx_release_workspace.argtypes = [vp]
        L.fglt_ctx_transform.restype = ctypes.c_int
        L.fglt_ctx_transform.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32,
                                         ctypes.c_int, ctypes.c_uint32, vp, vp,
                                         ctypes.POINTER(FgltStats), ctypes.POINTER(FgltError)]
        L.fglt_transform_csr32.restype = ctypes.c_int
        L.fglt_transform_csr32.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_uint32, vp, vp,
                                           ctypes.POINTER(FgltStats), ctypes.POINTER(FgltError)]
        L.fglt_net_from_raw.restype = ctypes.c_int
        L.fglt_net_from_raw.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int, vp,
                                        ctypes.POINTER(FgltError)]
        L.fglt_net_from_raw_matrix.restype = ctypes.c_int
        L.fglt_net_from_raw_matrix.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_uint32, vp,
                                               ctypes.c_int, vp, ctypes.POINTER(FgltError)]
        L.fglt_stage_prepare.restype = ctypes.c_int
        L.fglt_stage_prepare.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32,
                                         ctypes.c_int, ctypes.POINTER(FgltError)]
        L.fglt_stage_bounds.restype = ctypes.c_int
        L.fglt_stage_bounds.argtypes = [vp, ctypes.c_int, vp, ctypes.POINTER(FgltError)]
        L.fglt_stage_triangles.restype = ctypes.c_int
        L.fglt_stage_triangles.argtypes = [vp, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(FgltError)]
        L.fglt_stage_local.restype = ctypes.c_int
        L.fglt_stage_local.argtypes = [vp, ctypes.POINTER(FgltError)]
        L.fglt_stage_local_part.restype = ctypes.c_int
        L.fglt_stage_local_part.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(FgltError)]
        L.fglt_stage_roots.restype = ctypes.c_int
        L.fglt_stage_roots.argtypes = [vp, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.POINTER(ctypes.c_void_p),
                                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(FgltError)]
        L.fglt_stage_epilogue.restype = ctypes.c_int
        L.fglt_stage_epilogue.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, vp, vp,
                                          ctypes.POINTER(FgltError)]
        L.fglt_build_csr.restype = ctypes.c_int
        L.fglt_build_csr.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_uint32, vp, vp, vp, vp,
                                     ctypes.POINTER(FgltError)]
        L.fglt_csr_fetch.restype = ctypes.c_int
        L.fglt_csr_fetch.argtypes = [vp, vp, vp, ctypes.c_uint32, ctypes.POINTER(FgltError)]
        L.fglt_ctx_set_debug.restype = ctypes.c_int
        L.fglt_ctx_set_debug.argtypes = [vp, ctypes.c_int, ctypes.c_int]
        L.fglt_ctx_kernel_launches.restype = ctypes.c_uint64
        L.fglt_ctx_kernel_launches.argtypes = [vp]
        L.fglt_transform_multi.restype = ctypes.c_int
        L.fglt_transform_multi.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32,
                                           ctypes.c_int, vp, ctypes.c_int, ctypes.c_uint32, vp, vp,
                                           ctypes.POINTER(FgltStats), ctypes.POINTER(FgltError)]
        L.fglt_ctx_scratch_report.restype = ctypes.c_int
        L.fglt_ctx_scratch_report.argtypes = [vp, ctypes.c_char_p, ctypes.c_int]
        L.fglt_probe_smem_atomics.restype = ctypes.c_int
        L.fglt_probe_smem_atomics.argtypes = [vp, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(FgltError)]
        L.fglt_version.restype = ctypes.c_char_p
        L.fglt_version.argtypes = []
        L.fglt_device_count.restype = ctypes.c_int
        L.fglt_device_count.argtypes = []
        _lib = L
    return _lib


def dict_mask(ids) -> int:
    m = 3
    for i in ids:
        if not 0 <= int(i) < 16:
            raise ValueError(f"graphlet id {i} outside 0..15")
        m |= 1 << int(i)
    return m


def mask_ids(mask: int):
    mask |= 3
    return [i for i in range(16) if mask >> i & 1]


class TransformFailed(RuntimeError):
    def __init__(self, code, graphlet_id, vertex, msg):
        super().__init__(f"[{CODES.get(code, code)}] {msg}")
        self.code, self.graphlet_id, self.vertex, self.msg = code, graphlet_id, vertex, msg


def _raise(rc, err):
    raise TransformFailed(rc, err.graphlet_id, err.vertex, err.msg.decode(errors="replace"))


def transform_multi(rp: np.ndarray, ci: np.ndarray, devices, mask: int = 0xFFFF,
                    lenient=False):
    """fglt_transform_multi: host CSR in, host tables out, ranks on `devices`
    (repeats = the host-staged emulation of more ranks than GPUs)."""
    L = lib()
    rp = np.ascontiguousarray(rp, dtype=np.int32)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    n, nnz = len(rp) - 1, len(ci)
    k = len(mask_ids(mask))
    raw = np.empty((n, k), dtype=np.uint64)
    net = np.empty((n, k), dtype=np.uint64)
    dev = (ctypes.c_int * len(devices))(*devices)
    st, err = FgltStats(), FgltError()
    rc = L.fglt_transform_multi(rp.ctypes.data, ci.ctypes.data if nnz else None, n, nnz, mask,
                                int(lenient), dev, len(devices), 0, raw.ctypes.data,
                                net.ctypes.data, ctypes.byref(st), ctypes.byref(err))
    if rc:
        _raise(rc, err)
    return raw, net, st.as_dict()


class Context:
    """One device context (stream + cached workspace). ``stream`` is a raw
    cudaStream_t handle (e.g. ``torch.cuda.current_stream().cuda_stream``)."""

    def __init__(self, device: int = 0, stream: int = 0):
        self._L = lib()
        err = FgltError()
        self._h = self._L.fglt_ctx_create(device, ctypes.c_void_p(stream), ctypes.byref(err))
        if not self._h:
            _raise(err.code, err)

    def build_csr(self, eu, ev, n: int = 0, symmetrize=True, drop_self_loops=True, dedupe=True):
        """Device ingest (fglt_build_csr): undirected pairs -> sanitised int32 CSR."""
        eu = np.ascontiguousarray(eu, dtype=np.int64)
        ev = np.ascontiguousarray(ev, dtype=np.int64)
        out = np.zeros(4, dtype=np.int64)
        err = FgltError()
        rc = self._L.fglt_build_csr(self._h, eu.ctypes.data, ev.ctypes.data, len(eu), n,
                                    int(symmetrize), int(drop_self_loops), int(dedupe), 0,
                                    out[0:].ctypes.data, out[1:].ctypes.data,
                                    out[2:].ctypes.data, out[3:].ctypes.data, ctypes.byref(err))
        if rc:
            _raise(rc, err)
        n_out, nnz = int(out[0]), int(out[1])
        rp = np.empty(n_out + 1, dtype=np.int32)
        ci = np.empty(nnz, dtype=np.int32)
        rc = self._L.fglt_csr_fetch(self._h, rp.ctypes.data, ci.ctypes.data if nnz else None, 0,
                                    ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return rp, ci, {"self_loops_dropped": int(out[2]), "duplicates_merged": int(out[3])}

    def set_debug(self, key: int, value: int):
        rc = self._L.fglt_ctx_set_debug(self._h, key, value)
        if rc:
            raise ValueError(f"bad debug key {key}")

    def kernel_launches(self) -> int:
        return int(self._L.fglt_ctx_kernel_launches(self._h))

    def scratch_report(self):
        """{buffer: (bytes, staging)} of the last call (see fglt.h)."""
        buf = ctypes.create_string_buffer(1 << 14)
        self._L.fglt_ctx_scratch_report(self._h, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            f = line.split()
            out[f[0]] = (int(f[1]), len(f) > 2)
        return out

    def smem_atomic_rate(self) -> float:
        """Measured random shared-memory atomicAdd ops/s (on-chip roofline)."""
        out = ctypes.c_double(0)
        err = FgltError()
        rc = self._L.fglt_probe_smem_atomics(self._h, ctypes.byref(out), ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return float(out.value)

    def release_workspace(self):
        """Free the device workspace kept between calls (see include/fglt.h)."""
        rc = self._L.fglt_ctx_release_workspace(self._h)
        if rc:
            raise RuntimeError(f"fglt_ctx_release_workspace failed ({CODES.get(rc, rc)})")

    def close(self):
        if getattr(self, "_h", None):
            self._L.fglt_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def transform_host(self, rp: np.ndarray, ci: np.ndarray, mask: int = 0xFFFF, lenient=False,
                       timings=False, want_raw=True, want_net=True, raw=None, net=None):
        """Host CSR in, host tables out (H2D/D2H inside the call)."""
        rp = np.ascontiguousarray(rp, dtype=np.int32)
        ci = np.ascontiguousarray(ci, dtype=np.int32)
        n, nnz = len(rp) - 1, len(ci)
        k = len(mask_ids(mask))
        if want_raw and raw is None:
            raw = np.empty((n, k), dtype=np.uint64)
        if want_net and net is None:
            net = np.empty((n, k), dtype=np.uint64)
        st, err = FgltStats(), FgltError()
        flags = FGLT_TIMINGS if timings else 0
        rc = self._L.fglt_ctx_transform(self._h, rp.ctypes.data, ci.ctypes.data if nnz else None,
                                        n, nnz, mask, int(lenient), flags,
                                        raw.ctypes.data if want_raw else None,
                                        net.ctypes.data if want_net else None,
                                        ctypes.byref(st), ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return raw, net, st.as_dict()

    def transform_device(self, d_rp: int, d_ci: int, n: int, nnz: int, mask: int, d_raw: int,
                         d_net: int, lenient=False, timings=False):
        """Device pointers in and out (no host copies)."""
        st, err = FgltStats(), FgltError()
        flags = FGLT_INPUT_DEVICE | FGLT_OUTPUT_DEVICE | (FGLT_TIMINGS if timings else 0)
        rc = self._L.fglt_ctx_transform(self._h, d_rp, d_ci, n, nnz, mask, int(lenient), flags,
                                        d_raw or None, d_net or None, ctypes.byref(st),
                                        ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return st.as_dict()

    def transform_pinned(self, h_rp: int, h_ci: int, n: int, nnz: int, mask: int, h_raw: int,
                         h_net: int, lenient=False):
        """Host (pinned) pointers in and out: the e2e path of the C-ABI."""
        st, err = FgltStats(), FgltError()
        rc = self._L.fglt_ctx_transform(self._h, h_rp, h_ci, n, nnz, mask, int(lenient), 0,
                                        h_raw or None, h_net or None, ctypes.byref(st),
                                        ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return st.as_dict()

    def net_from_raw(self, raw: np.ndarray, mask: int, lenient=False, U=None):
        """net_from_raw on the device; U = the caller's k x k conversion matrix
        (None: U16(s,s))."""
        raw = np.ascontiguousarray(raw, dtype=np.uint64)
        net = np.empty_like(raw)
        err = FgltError()
        if U is None:
            rc = self._L.fglt_net_from_raw(self._h, raw.ctypes.data, raw.shape[0], mask,
                                           int(lenient), net.ctypes.data, ctypes.byref(err))
        else:
            U = np.ascontiguousarray(U, dtype=np.uint64)
            rc = self._L.fglt_net_from_raw_matrix(self._h, raw.ctypes.data, raw.shape[0], mask,
                                                  U.ctypes.data, int(lenient), net.ctypes.data,
                                                  ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return net

    # ---- staged (multi-rank) API
    def stage_prepare(self, d_rp: int, d_ci: int, n: int, nnz: int, mask: int, lenient=False):
        err = FgltError()
        rc = self._L.fglt_stage_prepare(self._h, d_rp, d_ci, n, nnz, mask, int(lenient),
                                        ctypes.byref(err))
        if rc:
            _raise(rc, err)

    def stage_bounds(self, world: int):
        b = np.zeros(world + 1, dtype=np.int64)
        err = FgltError()
        rc = self._L.fglt_stage_bounds(self._h, world, b.ctypes.data, ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return b

    def stage_triangles(self, u0: int, u1: int):
        p, cnt, err = ctypes.c_void_p(), ctypes.c_int64(), FgltError()
        rc = self._L.fglt_stage_triangles(self._h, u0, u1, ctypes.byref(p), ctypes.byref(cnt),
                                          ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return p.value or 0, cnt.value

    def stage_local(self):
        err = FgltError()
        rc = self._L.fglt_stage_local(self._h, ctypes.byref(err))
        if rc:
            _raise(rc, err)

    def stage_local_part(self, part: int, nparts: int, phase: int):
        """Row-partitioned vertex sweeps; phase 0 returns (device pointer, n)
        of the c3 vector to sum over ranks (count 0: nothing to sum)."""
        err = FgltError()
        p = ctypes.c_void_p()
        cnt = ctypes.c_int64()
        rc = self._L.fglt_stage_local_part(self._h, part, nparts, phase, ctypes.byref(p),
                                           ctypes.byref(cnt), ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return p.value or 0, cnt.value

    def stage_roots(self, u0: int, u1: int):
        p, cnt, err = ctypes.c_void_p(), ctypes.c_int64(), FgltError()
        rc = self._L.fglt_stage_roots(self._h, u0, u1, ctypes.byref(p), ctypes.byref(cnt),
                                      ctypes.byref(err))
        if rc:
            _raise(rc, err)
        return p.value or 0, cnt.value

    def stage_epilogue(self, v0: int, v1: int, d_raw: int, d_net: int):
        err = FgltError()
        rc = self._L.fglt_stage_epilogue(self._h, v0, v1, d_raw or None, d_net or None,
                                         ctypes.byref(err))
        return rc, err


def transform(rp, ci, ids=None, lenient=False, device=0):
    """One-shot host transform through the C-ABI (fglt_transform_csr32)."""
    L = lib()
    mask = 0xFFFF if ids is None else dict_mask(ids)
    rp = np.ascontiguousarray(rp, dtype=np.int32)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    n, nnz = len(rp) - 1, len(ci)
    k = len(mask_ids(mask))
    raw = np.empty((n, k), dtype=np.uint64)
    net = np.empty((n, k), dtype=np.uint64)
    st, err = FgltStats(), FgltError()
    rc = L.fglt_transform_csr32(rp.ctypes.data, ci.ctypes.data if nnz else None, n, nnz, mask,
                                int(lenient), device, 0, raw.ctypes.data, net.ctypes.data,
                                ctypes.byref(st), ctypes.byref(err))
    if rc:
        _raise(rc, err)
    return raw, net, st.as_dict()
