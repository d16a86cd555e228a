# A/B timing helper: build, run the GPU parity subset, time C5 (2^30 samples/GPU) twice.
set -e
python paper_2104_06311_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_upsample.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for i in 1 2; do python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --samples 1073741824 > gpurun_out/ab_$i.json 2>&1; done
for i in 1 2; do python -c "import json; d=json.loads(open('gpurun_out/ab_$i.json').read().strip().splitlines()[-1]); print(round(d['value'],2), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
