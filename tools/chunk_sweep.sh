# Call-size sweep on C5 (the full 2^32-sample stream per GPU): throughput vs samples per kk_process_frames call.
python paper_2104_06311_b200/build.py > /dev/null 2>&1
for c in 134217728 268435456 536870912 1073741824; do
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --chunk $c > gpurun_out/ab_c.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_c.json').read().strip().splitlines()[-1]); print($c, round(d['value'],2), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
done
