python paper_2104_06311_b200/build.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_upsample.py -q -x 2>&1 | tail -3
python bench.py --upsample 2 --samples 268435456 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k1u_t.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/k1u_t.json').read().strip().splitlines()[-1]); print(round(d['value'],2), {k:(round(v['avg_ms'],4), round(v['tflops'],1)) for k,v in d['kernels'].items()})"
