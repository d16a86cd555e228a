# K3 per-phase SM clocks (CTA 0, summed over its frames) from a -DKK_PHASE_TIMING build; diagnostic only.
KK_NVCC_DEFINES=-DKK_PHASE_TIMING python paper_2104_06311_b200/build.py --force > gpurun_out/phases_build.log 2>&1 || exit 1
python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep K3PHASES | tail -3 > gpurun_out/${1:-k3}_phases.txt
python paper_2104_06311_b200/build.py --force > /dev/null 2>&1
cat gpurun_out/${1:-k3}_phases.txt
