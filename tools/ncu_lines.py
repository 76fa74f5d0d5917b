"""Warp-stall samples aggregated per CUDA source line from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` (kernel built with -lineinfo).
usage: ncu_lines.py file.csv [top] [metric-column]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
col = hdr.index(sys.argv[3]) if len(sys.argv) > 3 else 4
lines = []
fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > col and r[0].isdigit() and r[col] not in ("-", ""):
        try:
            lines.append((float(r[col]), fname, int(r[0]), r[1].strip()))
        except ValueError:
            pass
tot = sum(v for v, *_ in lines)
print("column", hdr[col], "total", tot)
for v, f, ln, src in sorted(lines, reverse=True)[:top]:
    print("%6.1f%%  %s:%d  %s" % (100 * v / tot, f, ln, src[:110]))
