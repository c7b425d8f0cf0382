"""Summarise an ncu source page (--print-source=cuda,sass --csv) into the
hottest CUDA source lines by warp-stall samples. Dev tool."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0].isdigit():
        def num(x):
            try:
                return int(x)
            except ValueError:
                return 0
        out.append((num(r[4]), num(r[7]), cur, r[0], r[1][:100]))
tot = sum(o[0] for o in out) or 1
for o in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * o[0] / tot:5.1f}% inst {o[1]:12d} {o[2]}:{o[3]}  {o[4]}")
