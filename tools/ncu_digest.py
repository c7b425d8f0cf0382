"""Digest of one ncu --set full report: headline metrics, stall reasons and
the hottest source regions (dev tool). Usage: python tools/ncu_digest.py rep.ncu-rep [lines]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
print("kernel:", d.get("Kernel Name", ("?",))[0][:100])
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct"]:
    if k in d:
        print(f"  {k:60s} {d[k][0]} {d[k][1]}")
print("stalls (warps per issued instruction):")
for h, (v, u) in d.items():
    if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
        try:
            if float(v) > 0.1:
                print(f"  {h[34:-23]:22s} {float(v):.2f}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur = None
hdr = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r and r[0].isdigit() and len(r) > 10:
        def num(k):
            try:
                return float(r[hdr[k]])
            except (ValueError, KeyError):
                return 0.0
        out.append((num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"), cur, r[0], r[1][:80]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("hot lines: samples% inst% file:line")
for o in sorted(out, reverse=True)[:top]:
    print(f"  {100 * o[0] / ts:5.1f} {100 * o[1] / ti:5.1f}  {o[2]}:{o[3]}  {o[4]}")
