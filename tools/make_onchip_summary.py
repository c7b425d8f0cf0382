"""On-chip roofline of the dominant kernel from one `ncu --set full` capture:
raw-page CSV -> profiles/ncu_config<cfg>_dense_onchip.json (read by bench.py).
Usage: python tools/make_onchip_summary.py <raw.csv> <cfg> "<capture command>" """
import csv
import json
import sys

raw, cfg, source = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = list(csv.reader(open(raw)))
hdr, unit_row, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
unit_of = dict(zip(hdr, unit_row))


def f(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


units = {
    # every unit the kernel could be bound by, % of peak sustained over the launch
    "l1tex_data_pipe_lsu_wavefronts": f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    "l1tex_lsu_writeback": f("l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed"),
    "l1tex_to_xbar_requests": f("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    "sm_issue": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "sm_lsu_pipe": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed"),
    "l2": f("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    "dram": f("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
}
units = {k: v for k, v in units.items() if v is not None}
bound = max(units, key=units.get)
sh_w = f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
sh_c = f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
out = {
    "source": source, "config": cfg, "kernel": d.get("Kernel Name", "?")[:80],
    "duration_ms": (f("gpu__time_duration.sum") or 0) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit_of.get("gpu__time_duration.sum", "ms"), 1.0),
    "pct_of_peak": units, "bound": bound, "frac": units[bound] / 100.0,
    "shared_wavefronts": sh_w, "shared_bank_conflict_wavefronts": sh_c,
    "shared_atom_instructions": f("smsp__inst_executed_op_shared_atom.sum"),
    "shared_atom_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
    "global_load_requests": f("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    "global_load_sectors": f("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    "l2_hit_rate_pct": f("lts__t_sector_hit_rate.pct"),
    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "long_scoreboard_stall_per_issue": f("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
}
path = f"profiles/ncu_config{cfg}_dense_onchip.json"
json.dump(out, open(path, "w"), indent=1)
print(path, "bound:", bound, units[bound], "%")
