# A/B of K1's a4 exponent forms (K1_EXPV 0: __expf(a + ½ln I_ref); 1: log2 stored, ½ln2 on σ/1024; 2: ex2(fma)).
for n in ${VARS:-0 1 2}; do
  KK_NVCC_DEFINES="-DK1_EXPV=$n" python paper_2104_06311_b200/build.py --force > gpurun_out/build_$n.log 2>&1 || { echo build $n failed; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
  for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --samples 1073741824 > gpurun_out/abk1_${n}_$i.json 2>&1; done
  for i in 1 2; do python -c "import json; d=json.loads(open('gpurun_out/abk1_${n}_$i.json').read().strip().splitlines()[-1]); print('expv $n', round(d['value'],2), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
done
