# A/B timing of two source trees on one box: variant A = paper_2104_06311_b200/csrc (the working tree), variant B =
# the csrc directory given as $1 (e.g. a copy of the baseline made with `cp -r paper_2104_06311_b200/csrc
# scratch_ab/base` before editing). Each variant is built into its own library (KK_LIB) and benched alternately
# (ROUNDS rounds, default 3), ARGS passed to bench.py; prints per-kernel times. Diagnostic only.
B=${1:?usage: tools/ab_dirs.sh CSRC_DIR_B}
ARGS=${ARGS:---samples 1073741824 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline}
python paper_2104_06311_b200/build.py > gpurun_out/abA_build.log 2>&1 || { echo A build failed; exit 1; }
KK_CSRC=$B KK_LIB=/tmp/libkkrx_B.so KK_BUILD_DIR=/tmp/build_B python paper_2104_06311_b200/build.py > gpurun_out/abB_build.log 2>&1 || { echo B build failed; exit 1; }
for r in $(seq 1 ${ROUNDS:-3}); do
  for v in A B; do
    if [ $v = B ]; then export KK_LIB=/tmp/libkkrx_B.so; else unset KK_LIB; fi
    python bench.py $ARGS 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
  done
done
