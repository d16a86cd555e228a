# A/B of kernel variants on the upsampled (K1U) C5 path; see tools/ab_variants.sh.
set -e
CS=paper_2104_06311_b200/csrc
mkdir -p /tmp/ab_orig && cp $CS/* /tmp/ab_orig/
for v in ${@:-$(ls scratch_variants)}; do
  cp /tmp/ab_orig/* $CS/; cp scratch_variants/$v/* $CS/
  python paper_2104_06311_b200/build.py > /dev/null 2>&1
  for i in 1 2; do python bench.py --no-e2e --no-cpu-baseline --upsample 2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
done
cp /tmp/ab_orig/* $CS/; python paper_2104_06311_b200/build.py > /dev/null 2>&1
