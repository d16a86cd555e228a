"""Per CUDA source line: dynamic SASS opcode counts from `ncu --page source --csv --print-source cuda,sass`.
usage: python tools/ncu_sass_by_line.py X.csv OPCODE[,OPCODE] [norm] [top]"""
import csv
import re
import sys
from collections import defaultdict

path, ops = sys.argv[1], sys.argv[2].split(",")
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 8
rows = list(csv.reader(open(path)))
fname, cur = "?", None
agg = defaultdict(lambda: defaultdict(int))
src = {}
ie = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        ie = r.index("Instructions Executed")
        continue
    if ie is None or len(r) <= ie:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3].strip()) if len(r) > 3 else None
    if m and cur and r[ie].isdigit():
        agg[cur][m.group(2)] += int(r[ie])
for OP in ops:
    tot = sum(o.get(OP, 0) for o in agg.values())
    print(f"{OP}: {tot / norm:.1f}")
    for v, ln in sorted(((o.get(OP, 0), ln) for ln, o in agg.items()), reverse=True)[:top]:
        if v:
            print(f"   {v / norm:8.1f}  {ln[0][:12]}:{ln[1]:<4d} {src.get(ln, '')[:95]}")
