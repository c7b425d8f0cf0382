"""Row-block sharded FGlT across ranks (one process per GPU).

The graph is replicated (broadcast from rank 0); enumeration ROOTS (degree-
relabelled vertex ids) are split into contiguous blocks of equal exact work
(fglt_stage_bounds). The path has two genuine exchange steps, each one
collective over the process group (NCCL over NVLink on B200, gloo in the CPU
tests):

  1. all-reduce(sum) of the per-edge triangle counts C3 (uint32 per CSR slot)
     — every rank's roots contribute to edges it does not own;
  2. all-reduce(sum) of the per-vertex 4-cycle / diamond / 4-clique partials
     (3 x n uint64).

Then every rank runs the epilogue for its block of ORIGINAL vertex ids and
rank 0 gathers the rows. Integer sums are associative and commutative, so the
result is byte-identical for any world size (tests/test_dist_gloo.py,
tests/test_gpu_sharded.py).

The per-rank device work goes through a *stage backend*: ``CudaStages`` wraps
the C-ABI (include/fglt.h fglt_stage_*); tests substitute a numpy stand-in to
exercise this orchestration under gloo on CPU. There is no CPU fallback in the
product: CudaStages fails loudly without a device.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _capi


class _CAI:
    """Zero-copy __cuda_array_interface__ view of a device pointer."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}


def device_view(ptr: int, count: int, dtype: torch.dtype, device) -> torch.Tensor:
    typestr = {torch.int32: "<i4", torch.int64: "<i8"}[dtype]
    if count == 0:
        return torch.empty(0, dtype=dtype, device=device)
    return torch.as_tensor(_CAI(ptr, (count,), typestr), device=device)


class CudaStages:
    """Stage backend over the C-ABI on one CUDA device."""

    def __init__(self, device: torch.device, stream: torch.cuda.Stream | None = None):
        self.device = device
        self.stream = stream or torch.cuda.current_stream(device)
        self.ctx = _capi.Context(device.index or 0, self.stream.cuda_stream)

    def prepare(self, rp: torch.Tensor, ci: torch.Tensor, n: int, nnz: int, mask: int,
                lenient: bool):
        self.ctx.stage_prepare(rp.data_ptr(), ci.data_ptr() if nnz else 0, n, nnz, mask, lenient)

    def bounds(self, world: int) -> np.ndarray:
        return self.ctx.stage_bounds(world)

    def triangles(self, u0: int, u1: int) -> torch.Tensor:
        ptr, count = self.ctx.stage_triangles(u0, u1)
        return device_view(ptr, count, torch.int32, self.device)

    def local(self):
        self.ctx.stage_local()

    def local_part(self, part: int, nparts: int, phase: int) -> torch.Tensor:
        ptr, count = self.ctx.stage_local_part(part, nparts, phase)
        return device_view(ptr, count, torch.int64, self.device)

    def roots(self, u0: int, u1: int) -> torch.Tensor:
        ptr, count = self.ctx.stage_roots(u0, u1)
        return device_view(ptr, count, torch.int64, self.device)

    def epilogue(self, v0: int, v1: int, raw: torch.Tensor, net: torch.Tensor):
        rc, err = self.ctx.stage_epilogue(v0, v1, raw.data_ptr() if raw.numel() else 0,
                                          net.data_ptr() if net.numel() else 0)
        return rc, (err.code, err.graphlet_id, err.vertex, err.msg.decode(errors="replace"),
                    int(err.order_key))


def row_blocks(n: int, world: int):
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


def sharded_transform(stages, rp: torch.Tensor | None, ci: torch.Tensor | None, n: int, nnz: int,
                      mask: int = 0xFFFF, lenient: bool = False, group=None, root: int = 0):
    """Run the sharded transform. ``rp``/``ci`` must be valid on ``root`` and
    pre-allocated (any content) with the right sizes on the other ranks.
    Returns (raw, net) tensors of shape (n, k) on ``root`` and None elsewhere.
    Raises _capi.TransformFailed with the lowest-ordered failure of any rank."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    device = rp.device
    k = len(_capi.mask_ids(mask))
    # the CSR is replicated (input lives on root)
    dist.broadcast(rp, src=root, group=group)
    if nnz:
        dist.broadcast(ci, src=root, group=group)
    stages.prepare(rp, ci, n, nnz, mask, lenient)
    b = stages.bounds(world)
    u0, u1 = int(b[rank]), int(b[rank + 1])
    # exchange 1: per-edge triangle counts
    c3 = stages.triangles(u0, u1)
    if c3.numel() and world > 1:
        dist.all_reduce(c3, op=dist.ReduceOp.SUM, group=group)
    # vertex sweeps on my rows (r = rank mod world) only; sweep C reads every
    # row's c3, so the c3 vector is summed in between (exchange 1b, n values)
    c3v = stages.local_part(rank, world, 0)
    if c3v.numel() and world > 1:
        dist.all_reduce(c3v, op=dist.ReduceOp.SUM, group=group)
    stages.local_part(rank, world, 1)
    # exchange 2: per-vertex partials (world > 1: d14 d10 p3 d9 of my rows and
    # c4 d13 d15 of my roots, 7n values; world 1: nothing to sum)
    vec = stages.roots(u0, u1)
    if vec.numel() and world > 1:
        dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
    # epilogue on my block of original ids, then gather to root
    blocks = row_blocks(n, world)
    v0, v1 = blocks[rank]
    rows = max(hi - lo for lo, hi in blocks) if n else 0
    raw = torch.zeros((rows, k), dtype=torch.int64, device=device)
    net = torch.zeros((rows, k), dtype=torch.int64, device=device)
    rc, err = stages.epilogue(v0, v1, raw[: v1 - v0], net[: v1 - v0])
    # combine failures: the reference reports the first in (stage, vertex) order
    none = torch.iinfo(torch.int64).max
    keyu = torch.tensor([err[4] if rc else none], dtype=torch.int64, device=device)
    dist.all_reduce(keyu, op=dist.ReduceOp.MIN, group=group)
    if keyu.item() != none:
        best = int(keyu.item())
        mine = bool(rc) and err[4] == best
        code_tensor = torch.tensor([rc if mine else -1, err[1] if mine else -1,
                                    err[2] if mine else -1], dtype=torch.int64, device=device)
        dist.all_reduce(code_tensor, op=dist.ReduceOp.MAX, group=group)
        code, g, v = (int(x) for x in code_tensor.tolist())
        raise _capi.TransformFailed(code, g, v, f"rank-combined failure (order key {best:#x})")
    if world == 1:
        return raw[:n], net[:n]
    if rank == root:
        raw_parts = [torch.empty_like(raw) for _ in range(world)]
        net_parts = [torch.empty_like(net) for _ in range(world)]
    else:
        raw_parts = net_parts = None
    dist.gather(raw, raw_parts, dst=root, group=group)
    dist.gather(net, net_parts, dst=root, group=group)
    if rank != root:
        return None, None
    raw_out = torch.cat([p[: hi - lo] for p, (lo, hi) in zip(raw_parts, blocks)])
    net_out = torch.cat([p[: hi - lo] for p, (lo, hi) in zip(net_parts, blocks)])
    return raw_out, net_out
