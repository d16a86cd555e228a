# Per-configuration bench lines (BASELINE.json configs C1–C5) + variants, final code of the round.
set -e
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
mkdir -p gpurun_out/cfg
python bench.py --workload C1 --samples 65536 --steps 20 --warmup 5 --no-e2e --cpu-frames 4 > gpurun_out/cfg/C1.json 2>&1
python bench.py --workload C2 --samples 4194304 --steps 10 --warmup 3 --no-e2e --cpu-frames 32 > gpurun_out/cfg/C2.json 2>&1
python bench.py --workload C3 --samples 16777216 --steps 10 --warmup 3 --no-e2e --cpu-frames 32 > gpurun_out/cfg/C3.json 2>&1
python bench.py --workload C4 --samples 67108864 --steps 5 --warmup 3 --no-e2e --cpu-frames 32 > gpurun_out/cfg/C4.json 2>&1
python bench.py --workload C5 --steps 5 --warmup 3 --cpu-frames 64 > gpurun_out/cfg/C5.json 2>&1
python bench.py --workload C5 --steps 3 --warmup 3 --upsample 2 --no-e2e --cpu-frames 32 > gpurun_out/cfg/C5_up2.json 2>&1
python bench.py --workload C5 --steps 3 --warmup 3 --static-cd --no-e2e --cpu-frames 32 > gpurun_out/cfg/C5_scd.json 2>&1
python bench.py --workload C4 --samples 67108864 --steps 5 --warmup 3 --static-cd --no-e2e --cpu-frames 32 > gpurun_out/cfg/C4_scd.json 2>&1
python bench.py --workload C5 --steps 3 --warmup 3 --eq-mode ddlms --no-e2e --cpu-frames 32 > gpurun_out/cfg/C5_ddlms.json 2>&1
for f in C1 C2 C3 C4 C5 C5_up2 C5_scd C4_scd C5_ddlms; do python -c "
import json; d=json.loads(open('gpurun_out/cfg/$f.json').read().strip().splitlines()[-1])
k=d['kernels']; c=d['cpu_baseline'] or {}
print('$f', round(d['value'],2), {n:(round(v['avg_ms']*1e3,1), round(v['tflops'],1)) for n,v in k.items()}, 'frac', round(d['roofline']['frac'],3), 'cpu', c.get('value'), c.get('cores'), 'parity', c.get('parity_decisions_identical'), 'e2e', (d['e2e'] or {}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
