# Default C5 bench + the two variant arrangements (KK upsampling, paper DDLMS), kernel times per line.
python paper_2104_06311_b200/build.py > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for a in "" "--upsample 2" "--eq-mode ddlms"; do
  python bench.py --no-e2e --no-cpu-baseline $a 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$a]', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
