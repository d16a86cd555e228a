# Functional smoke of bench.py's N > 1 path on ONE GPU (two ranks share it; gloo process group). Numbers from
# such a run are meaningless and never reported — it only checks that the multi-rank code path runs.
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 2 --warmup 1 --samples 268435456 --dist-backend gloo > gpurun_out/mr_bench.json 2> gpurun_out/mr_bench.err
echo "bench rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "ref rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 2 --steps 2 --warmup 1 --samples 268435456 --dist-backend gloo --ingest single --no-cpu-baseline > gpurun_out/mr_single.json 2> gpurun_out/mr_single.err
echo "single rc=$?"
