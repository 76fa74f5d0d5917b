"""Per-source-line stall samples and executed instructions from `ncu --page source --csv --print-source cuda,sass`.
usage: ncu_lines2.py src.csv [top]"""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = None; hdr = None; cur = None
samp = collections.Counter(); inst = collections.Counter(); fp = collections.Counter(); src = {}
tot_s = 0
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr is None or len(r) < 8: continue
    if r[0] != '':
        cur = (cur_file, int(r[0])); src[cur] = r[1].strip()[:100]; continue
    ins = r[3].strip()
    try: s = int(r[4]); n = int(r[7])
    except ValueError: continue
    samp[cur] += s; inst[cur] += n; tot_s += s
    op = re.match(r'(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)', ins)
    if op and op.group(1) in ('DFMA', 'DMUL', 'DADD', 'DSETP', 'DMMA'): fp[cur] += n
print('total samples', tot_s, 'instructions', sum(inst.values()), 'fp64', sum(fp.values()))
for k, v in samp.most_common(top):
    print('%5.1f%%  inst %9d  fp64 %9d  %s:%d  %s' % (100 * v / tot_s, inst[k], fp[k], k[0], k[1], src.get(k, '')))
