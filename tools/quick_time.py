"""Quick device timing of the transform on one config (dev tool)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2007_11111_b200 import _capi, graphs

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t0 = time.time()
name, rp, ci = graphs.config(cfg)
print(name, "n", len(rp) - 1, "m", len(ci) // 2, "gen", round(time.time() - t0, 2), "s", flush=True)
dev = torch.device("cuda:0")
s = torch.cuda.Stream()
ctx = _capi.Context(0, s.cuda_stream)
d_rp = torch.from_numpy(rp).to(dev)
d_ci = torch.from_numpy(ci).to(dev)
n, nnz = len(rp) - 1, len(ci)
raw = torch.empty((n, 16), dtype=torch.int64, device=dev)
net = torch.empty((n, 16), dtype=torch.int64, device=dev)
for it in range(4):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        st = ctx.transform_device(d_rp.data_ptr(), d_ci.data_ptr(), n, nnz, 0xFFFF, raw.data_ptr(), net.data_ptr(), timings=(it == 3))
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"iter {it}: {ms:.3f} ms  -> {n and (nnz//2)/ms/1e3:.3e} edges/s", flush=True)
import hashlib
h = hashlib.sha256(raw.cpu().numpy().tobytes() + net.cpu().numpy().tobytes()).hexdigest()[:16]
print("sha", h)
print(json.dumps(st))
