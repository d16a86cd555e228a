# Build, GPU test suite, smoke and one default bench line (TAG names the outputs under gpurun_out/).
TAG=${1:-chk}
python paper_2104_06311_b200/build.py > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 2), "clocks", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
print({k: round(v["avg_ms"], 4) for k, v in d["kernels"].items()}, "frac", round(d["roofline"]["frac"], 3), "e2e", (d.get("e2e") or {}).get("value"))
PY
