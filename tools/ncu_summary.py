"""Summarise an ncu report (--set full) and a launch-list CSV into markdown + the bench's traffic file.

usage: python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT.md [TRAFFIC.json]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "DRAM read (MB)"),
    ("dram__bytes_write.sum", "DRAM write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn. smem / CTA (KB)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def main(report, launches, out_md, traffic_json=None):
    hdr, units, data = raw(report)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary — `{report}`", "", "Captured with `ncu --set full --clock-control none --import-source on`"
             " on one B200 (bench.py --samples 2^28, one 2^28-sample call per kernel). Values per launch.", ""]
    names = [r[col["Kernel Name"]].split("(")[0].replace("void ", "") for r in data]
    lines.append("| metric | " + " | ".join(names) + " |")
    lines.append("|---|" + "---|" * len(names))
    traffic = {}
    for m, label in METRICS:
        if m not in col:
            continue
        vals = [r[col[m]] for r in data]
        lines.append(f"| {label} (`{m}`, {units[col[m]]}) | " + " | ".join(vals) + " |")
    for r, n in zip(data, names):
        try:
            rd = float(r[col["dram__bytes_read.sum"]].replace(",", ""))
            wr = float(r[col["dram__bytes_write.sum"]].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[col["dram__bytes_read.sum"]], 1)
            key = "K1u_kk" if "k1u_" in n else "K1_kk" if "k1_" in n else "K2_mf" if "k2_" in n else "K3_eq" if ("k3_" in n or "k3s_" in n) else n
            traffic[key] = traffic.get(key, 0.0) + (rd + wr) * scale   # K3 = K3a + K3s + K3c
        except (KeyError, ValueError):
            pass
    # launch list shares
    tot = defaultdict(float)
    cnt = defaultdict(int)
    if launches:
        txt = open(launches).read().splitlines()
        start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
        for r in csv.DictReader(io.StringIO("\n".join(txt[start:]))):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            n = r["Kernel Name"].split("(")[0].replace("void ", "")
            v = float(r["Metric Value"].replace(",", ""))
            tot[n] += v
            cnt[n] += 1
        ours = {k: v for k, v in tot.items() if k.split("<")[0].split("::")[-1].startswith(("k1_", "k2_", "k3_", "k3s_"))}
        s = sum(ours.values())
        lines += ["", "## Launch list (ncu `gpu__time_duration.sum`, cold-cache, serialised)", "",
                  "| kernel | launches | total (us) | share of K1+K2+K3 |", "|---|---|---|---|"]
        for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / s:.1%} |")
        other = sum(tot.values()) - s
        lines.append(f"| (torch generator / copy kernels, outside the timed region) | "
                     f"{sum(cnt.values()) - sum(cnt[k] for k in ours)} | {other / 1e3:.1f} | — |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    if traffic_json:
        json.dump({"source": report, "chunk_samples": int(os.environ.get("KK_NCU_CHUNK", 1 << 28)), "bytes_per_launch": traffic}, open(traffic_json, "w"),
                  indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "/dev/stdout",
         sys.argv[4] if len(sys.argv) > 4 else None)
