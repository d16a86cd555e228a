# K1U (upsample = 2) ncu capture at the bench's 2^28-sample calls; plain run first.
set -e
python paper_2104_06311_b200/build.py > gpurun_out/build.log 2>&1
python bench.py --upsample 2 --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/k1u_plain.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k1u_kk" -c 1 -o gpurun_out/${1:-k1u_s2} \
    python bench.py --upsample 2 --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/k1u_full.log 2>&1
echo done
