"""Quick summary of a one-kernel ncu --set full report: throughputs, stall ratios, smem wavefronts, dynamic
opcode mix. usage: python tools/ncu_k3_quick.py REPORT.ncu-rep [frames_per_launch] [kernel regex [launch skip]]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 16384.0
kern = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
if len(sys.argv) > 4:
    kern += ["--launch-skip", sys.argv[4], "--launch-count", "1"]


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep] + kern + list(a), capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
d = dict(zip(rows[0], rows[2]))
for k in ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
          "l1tex__throughput.avg.pct_of_peak_sustained_active"]:
    v = d.get(k)
    print(f"{k:70s} {v}")
print("per frame: warp inst %.0f, smem wavefronts %.0f" % (float(d["smsp__inst_executed.sum"]) / frames,
                                                          float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]) / frames))
st = {k: float(v or 0) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")}
print("stalls/issue:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:9]))
srows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hdr = srows[1]
ie = hdr.index("Instructions Executed")
agg = defaultdict(int)
seen = set()
for r in srows[2:]:
    if len(r) <= ie or not r[ie].isdigit() or r[0] in seen:   # the page lists every address twice: count once
        continue
    seen.add(r[0])
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[1].strip())
    if m:
        agg[m.group(2)] += int(r[ie])
T = sum(agg.values())
print("opcodes per frame per warp (8 warps):", ", ".join(f"{k} {v / frames / 8:.0f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:22]))
