set -e
python paper_2104_06311_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "ddlms or dd_ or guarded or ingest" 2>&1 | tail -3
for i in 1 2; do python bench.py --eq-mode ddlms --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --samples 1073741824 > gpurun_out/ab_dd.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/ab_dd.json').read().strip().splitlines()[-1]); print(round(d['value'],2), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()}, d['quality']['per_format'])"; done
