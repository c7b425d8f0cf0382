"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes)
per kernel name. Usage: python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import json
import sys


def summarize(path, top=16, as_json=False):
    rows = list(csv.reader(open(path)))
    start = hdr = None
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    idx = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[start:]:
        if len(r) < len(hdr):
            continue
        name = r[idx["Kernel Name"]]
        name = name.split("(")[0]
        met, unit = r[idx["Metric Name"]], r[idx["Metric Unit"]]
        val = float(r[idx["Metric Value"]].replace(",", ""))
        a = agg.setdefault(name, {"launches": 0, "us": 0.0, "dram_read": 0.0, "dram_write": 0.0,
                                  "l2_sectors": 0.0, "l2_hit_sectors": 0.0})
        if met == "gpu__time_duration.sum":
            a["launches"] += 1
            a["us"] += val * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
        elif met == "dram__bytes_read.sum":
            a["dram_read"] += val * scale.get(unit, 1)
        elif met == "dram__bytes_write.sum":
            a["dram_write"] += val * scale.get(unit, 1)
        elif met == "lts__t_sectors.sum":
            a["l2_sectors"] += val
        elif met == "lts__t_sectors_lookup_hit.sum":
            a["l2_hit_sectors"] += val
    tot = sum(a["us"] for a in agg.values())
    for a in agg.values():  # L2 hit rate over the kernel's launches (when the list has the sectors)
        sec, hit = a.pop("l2_sectors"), a.pop("l2_hit_sectors")
        a["l2_hit_rate"] = hit / sec if sec else None
    items = sorted(agg.items(), key=lambda kv: -kv[1]["us"])
    if as_json:
        return {"total_us": tot, "dram_bytes": sum(a["dram_read"] + a["dram_write"] for a in agg.values()),
                "kernels": [{"name": k, **v, "share": v["us"] / tot} for k, v in items]}
    for k, a in items[:top]:
        print(f"{a['us'] / 1e3:9.3f} ms {100 * a['us'] / tot:5.1f}% x{a['launches']:3d} "
              f"rd {a['dram_read'] / 1e9:7.3f} GB wr {a['dram_write'] / 1e9:6.3f} GB "
              f"L2hit {('%4.0f%%' % (100 * a['l2_hit_rate'])) if a['l2_hit_rate'] is not None else '   - '}  {k[:70]}")
    print(f"total {tot / 1e3:.3f} ms  dram {sum(a['dram_read'] + a['dram_write'] for a in agg.values()) / 1e9:.3f} GB")


if __name__ == "__main__":
    summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 16)
