# A/B kernel variants: scratch_variants/<name>/<file> replaces paper_2104_06311_b200/csrc/<file>; each variant is
# built and benched (kernel times), then the original sources are restored. Diagnostic only.
set -e
CS=paper_2104_06311_b200/csrc
mkdir -p /tmp/ab_orig && cp $CS/* /tmp/ab_orig/
for v in ${@:-$(ls scratch_variants)}; do
  cp /tmp/ab_orig/* $CS/
  cp scratch_variants/$v/* $CS/
  python paper_2104_06311_b200/build.py > gpurun_out/ab_build_$v.log 2>&1 || { echo "$v build failed"; continue; }
  for i in 1 2; do
    python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
  done
done
cp /tmp/ab_orig/* $CS/
python paper_2104_06311_b200/build.py > /dev/null 2>&1
