# Per-kernel device times of one bench configuration (ncu launch list, serialised and cold-cache — shares, not
# absolutes): tools/launch_times.sh TAG [bench args]
TAG=${1:-lt}; shift
python paper_2104_06311_b200/build.py > /dev/null 2>&1 || exit 1
ARGS=${@:---samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k2|k3" --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > /dev/null 2>&1
python - <<PY
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/${TAG}_launches.csv")) if len(r) > 10]
h = rows[0]; kn = h.index("Kernel Name"); mv = h.index("Metric Value")
t = collections.defaultdict(list)
for r in rows[1:]:
    t[r[kn].split("(")[0]].append(float(r[mv].replace(",", "")))
tot = sum(sum(v) for v in t.values())
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} n={len(v):3d} avg={sum(v)/len(v)/1e3:9.1f} us share={sum(v)/tot*100:5.1f}%")
PY
