# A/B of K2's resident CTAs per SM (K2_CTAS_4096 = 4, 5, 6): rebuild, bench C5 at 2^30 samples/GPU twice each.
for n in ${CTAS:-4 5 6}; do
  KK_NVCC_DEFINES="-DK2_CTAS_4096=$n" python paper_2104_06311_b200/build.py --force > gpurun_out/build_$n.log 2>&1 || { echo build $n failed; continue; }
  for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --samples 1073741824 > gpurun_out/abk2_${n}_$i.json 2>&1; done
  for i in 1 2; do python -c "import json; d=json.loads(open('gpurun_out/abk2_${n}_$i.json').read().strip().splitlines()[-1]); print('ctas $n', round(d['value'],2), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items()})"; done
done
