"""Print selected raw metrics per launch from an `ncu --page raw --csv` dump. Dev tool."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
idx = {x: i for i, x in enumerate(h)}
pats = sys.argv[2:] or ["gpu__time_duration.sum", "throughput.avg.pct", "stalled", "op_red", "op_atom"]
for name in h:
    if any(p in name for p in pats):
        vals = [r[idx[name]] for r in rows[2:]]
        print(name[:70].ljust(72), rows[1][idx[name]][:8].ljust(8), " ".join(v[:9].rjust(9) for v in vals))
