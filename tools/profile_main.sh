# Main-path profile refresh (one gpurun call; each ncu command preceded by its plain run). TAG names the outputs.
set -e
TAG=${1:-r02}
python paper_2104_06311_b200/build.py > gpurun_out/build.log 2>&1
python bench.py --steps 2 --warmup 1 > gpurun_out/${TAG}_prof_bench_plain.json 2> gpurun_out/${TAG}_prof_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_kk|k2_mf|k3" -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${TAG}_prof_launch.log 2>&1
python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_prof_small_plain.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k1_kk|k2_mf|k3" -c 5 -o gpurun_out/${TAG}_full -f \
    python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_prof_full.log 2>&1
echo done
