"""One warm-up transform, then one transform inside an NVTX range "step" —
the command the ncu launch list / --set full captures are taken on:

  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum ... python tools/profile_step.py 3
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_11111_b200 import _capi, graphs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
name, rp, ci = graphs.config(cfg)
dev = torch.device("cuda:0")
s = torch.cuda.Stream()
ctx = _capi.Context(0, s.cuda_stream)
d_rp = torch.from_numpy(rp).to(dev)
d_ci = torch.from_numpy(ci).to(dev)
n, nnz = len(rp) - 1, len(ci)
raw = torch.empty((n, 16), dtype=torch.int64, device=dev)
net = torch.empty((n, 16), dtype=torch.int64, device=dev)
torch.cuda.synchronize()
ctx.transform_device(d_rp.data_ptr(), d_ci.data_ptr(), n, nnz, 0xFFFF, raw.data_ptr(), net.data_ptr())
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
st = ctx.transform_device(d_rp.data_ptr(), d_ci.data_ptr(), n, nnz, 0xFFFF, raw.data_ptr(), net.data_ptr())
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(name, "launches per step", st["kernel_launches"])
