# Repeat the default bench N times (kernel times per run) — run-to-run variance check.
python paper_2104_06311_b200/build.py > /dev/null 2>&1 || exit 1
for i in $(seq 1 ${1:-3}); do
  python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
done
