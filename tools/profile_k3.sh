# K3 deep profile (one gpurun call): plain run, then one ncu --set full capture of a single K3 launch, then the
# per-phase clock breakdown (-DKK_PHASE_TIMING build; diagnostic only). TAG names the outputs.
TAG=${1:-k3}
python paper_2104_06311_b200/build.py > gpurun_out/${TAG}_build.log 2>&1 || exit 1
python bench.py --samples 268435456 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_plain.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-k3}" -s ${SKIP:-0} -c ${COUNT:-3} -o gpurun_out/${TAG} -f \
    python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
if [ -n "$PHASES" ]; then bash tools/k3_phases.sh ${TAG}; fi
