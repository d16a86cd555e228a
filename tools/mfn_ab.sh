python paper_2104_06311_b200/build.py > /dev/null 2>&1
for n in 4096 8192; do python bench.py --no-e2e --no-cpu-baseline --mf-n $n 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
