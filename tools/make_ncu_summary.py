"""Build profiles/ncu_config<k>_summary.json from an ncu --csv launch list
(gpu__time_duration.sum, dram__bytes_read/write.sum per launch of ONE step,
tools/profile_step.py inside the NVTX range "step"). bench.py reads it for
roofline.traffic. Usage: python tools/make_ncu_summary.py launches.csv CFG "ncu command"
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_summary import summarize  # noqa: E402

csv_path, cfg, cmd = sys.argv[1], int(sys.argv[2]), sys.argv[3]
s = summarize(csv_path, as_json=True)
out = {"source": cmd, "config": cfg, "dram_bytes_per_step": s["dram_bytes"],
       "kernel_time_sum_us": s["total_us"], "kernels": s["kernels"]}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", f"ncu_config{cfg}_summary.json"), "w") as f:
    json.dump(out, f, indent=1)
print(f"config {cfg}: {s['total_us'] / 1e3:.2f} ms kernel sum, {s['dram_bytes'] / 1e9:.3f} GB DRAM")
