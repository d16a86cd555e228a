"""The multi-rank product path on the GPU: bench.py's strong sharding of one stream
(shard.plan_strong, BASELINE configs[4]) run as two ranks sharing cuda:0 over a gloo group (the pool gives one
GPU per call; the counter allreduce is host-staged, the kernels are the same), against the single-rank run of
the same stream: the allreduced error counters must be bit-identical (P13: every grid is anchored at global
sample 0, so shards + halos reproduce the single-GPU decisions). Timings of this run are meaningless."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--samples", str(1 << 24), "--chunk", str(1 << 22), "--steps", "1", "--warmup", "1", "--no-e2e",
        "--no-cpu-baseline"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_two_rank_strong_sharding_counts_equal_single_rank():
    one = subprocess.run([sys.executable, "bench.py", "--gpus", "1"] + ARGS, cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-3000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                          "--dist-backend", "gloo"] + ARGS, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert two.returncode == 0, two.stderr[-3000:]
    a, b = _line(one.stdout), _line(two.stdout)
    assert a["scaling"] == b["scaling"] == "strong" and b["n_gpus"] == 2
    assert b["dist"]["world_size"] == 2 and [r["rank"] for r in b["dist"]["ranks"]] == [0, 1]
    sh = b["dist"]["ranks"]
    assert sh[0]["shard_first"] == 0 and sh[1]["shard_first"] == sh[0]["shard_samples"]
    assert sh[0]["shard_samples"] + sh[1]["shard_samples"] == 1 << 24
    assert a["quality"]["counts"] == b["quality"]["counts"]
    assert a["quality"]["frames"] == b["quality"]["frames"] == (1 << 24) // 16384
    assert sum(a["quality"]["counts"]["bit_err"]) > 0                   # non-trivial counts (64-QAM errors)
