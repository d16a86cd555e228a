# K3 per-phase clocks (CTA 0) of the working tree (A) and of the csrc directory $1 (B); diagnostic builds with
# -DKK_PHASE_TIMING into /tmp (the in-tree library is untouched).
B=${1:?usage: tools/ab_phases.sh CSRC_DIR_B}
for v in A B; do
  if [ $v = A ]; then SRC=paper_2104_06311_b200/csrc; else SRC=$B; fi
  KK_NVCC_DEFINES=-DKK_PHASE_TIMING KK_CSRC=$SRC KK_LIB=/tmp/libkkrx_ph$v.so KK_BUILD_DIR=/tmp/build_ph$v \
    python paper_2104_06311_b200/build.py > gpurun_out/ph${v}_build.log 2>&1 || { echo $v build failed; exit 1; }
  KK_LIB=/tmp/libkkrx_ph$v.so python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 \
    | grep K3PHASES | tail -1 | sed "s/^/$v /"
done
