"""Aggregate an ncu `--page source --print-source cuda,sass --csv` export by CUDA source line.

usage: ncu -i prof.ncu-rep --page source --csv --kernel-name regex:K --print-source cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hi]
    fname = "?"
    col = {h: i for i, h in enumerate(hdr)}
    samp = hdr.index("Warp Stall Sampling (All Samples)")
    inst = hdr.index("Instructions Executed")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = defaultdict(lambda: defaultdict(float))
    src = {}
    line = None
    total = 0.0
    for r in rows[hi + 1:]:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            line = None
            continue
        if len(r) < len(hdr) or r[0] == "Line No":
            continue
        if r[0]:
            line = (fname, int(r[0]))
            src[line] = r[1].strip()
        if line is None:
            continue
        try:
            s = float(r[samp] or 0)
        except ValueError:
            continue
        total += s
        a = agg[line]
        a["samples"] += s
        a["inst"] += float(r[inst] or 0)
        for st in stalls:
            a[st] += float(r[col[st]] or 0)
    print(f"total stall samples {total:.0f}")
    for ln, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        top_st = sorted(((a[s], s[6:]) for s in stalls), reverse=True)[:3]
        st = ", ".join(f"{n}:{v / max(a['samples'], 1):.0%}" for v, n in top_st if v)
        print(f"{a['samples'] / total:6.1%} {ln[0][:10]}:{ln[1]:<4d} inst {a['inst']:11.0f}  [{st}]  {src.get(ln, '')[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
