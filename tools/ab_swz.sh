set -e
CS=paper_2104_06311_b200/csrc
mkdir -p /tmp/ab_orig && cp $CS/* /tmp/ab_orig/
for v in head swz; do
  cp /tmp/ab_orig/* $CS/; cp scratch_variants/$v/* $CS/
  python paper_2104_06311_b200/build.py > /dev/null 2>&1
  for a in "" "--upsample 2"; do python bench.py --no-e2e --no-cpu-baseline $a 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v [$a]', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
done
cp /tmp/ab_orig/* $CS/; python paper_2104_06311_b200/build.py > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_upsample.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
