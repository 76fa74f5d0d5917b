"""Top SASS instructions by a stall reason from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
data = rows[2:]
tot = sum(float(r[ix[reason]] or 0) for r in data)
allsamp = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(reason, "total", tot, "of all samples", allsamp)
top = sorted(range(len(data)), key=lambda i: -float(data[i][ix[reason]] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]
for i in top:
    r = data[i]
    # show the instruction and the 2 preceding ones
    print("%6s  %5d  %s" % (r[ix[reason]], i, r[ix["Source"]].strip()))
