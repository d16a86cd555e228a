# Time several csrc variants on one box (diagnostic): tools/ab_multi.sh DIR1 DIR2 ... ; the working tree is "A".
ARGS=${ARGS:---samples 1073741824 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline}
python paper_2104_06311_b200/build.py > /dev/null 2>&1 || { echo A build failed; exit 1; }
i=0
for d in "$@"; do
  i=$((i+1))
  KK_CSRC=$d KK_LIB=/tmp/libkk_v$i.so KK_BUILD_DIR=/tmp/build_v$i python paper_2104_06311_b200/build.py > /tmp/build_v$i.log 2>&1 || { echo "$d build failed"; tail -5 /tmp/build_v$i.log; }
done
for r in $(seq 1 ${ROUNDS:-2}); do
  unset KK_LIB
  python bench.py $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
  i=0
  for d in "$@"; do
    i=$((i+1))
    KK_LIB=/tmp/libkk_v$i.so python bench.py $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', round(d['value'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items()})"
  done
done
