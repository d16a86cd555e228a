# Main-path profile refresh at the current code (TAG = report name under gpurun_out/).
# Each ncu command is preceded by its plain run (exit 0 without ncu first).
set -e
TAG=${1:-r01_head}
python paper_2104_06311_b200/build.py > gpurun_out/build.log 2>&1
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_kk|k2_mf|k3_eq" -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_launch.log 2>&1
python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_small_plain.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k1_kk|k2_mf|k3_eq" -c 3 -o gpurun_out/${TAG} \
    python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_full.log 2>&1
echo done
