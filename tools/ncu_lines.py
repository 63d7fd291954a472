"""Per-source-line instruction / stall breakdown of an ncu capture
(`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv`).
python tools/ncu_lines.py X.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 26
cur_file = cur_line = hdr = None
agg = defaultdict(lambda: [0, 0, 0])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split('/')[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        iss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0] == "Function Name":
        continue
    if r[0] != '':
        cur_line = (cur_file, int(r[0]), r[1][:100])
        continue
    if hdr is None or len(r) <= ie:
        continue
    try:
        n, s = int(r[ie]), int(r[iss])
    except ValueError:
        continue
    a = agg[cur_line]
    a[0] += n
    a[1] += s
    if 'IMAD' in r[3]:
        a[2] += n
tot = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*v[0]/tot:5.1f}% imad {100*v[2]/tot:4.1f}% stall {100*v[1]/ts:4.1f}%  {k[0]}:{k[1]} {k[2]}")
