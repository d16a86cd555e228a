"""Single-ingest delivery on the GPU path (paper_2104_06311_b200/ingest.py): windows staged from
pinned host memory on the side stream, double-buffered, processed by kk_process_frames on the caller's stream —
decisions and counters bit-identical to processing the device-resident stream directly (world size 1 here;
the multi-rank delivery is covered with gloo in tests/test_multi_rank.py)."""
import pytest
import torch

from gpu_case import make_case, receiver_for

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2104_06311_b200 import ingest, shard  # noqa: E402

F = 16384


@pytest.mark.parametrize("upsample", [1, 2])
def test_single_ingest_matches_direct(upsample):
    n, chunk = 6 * F, 2 * F
    case = make_case(M=16, dl=112000.0, cspr=10.0, esn0=17.0, n=n, first=3 * F, seed=131, upsample=upsample)
    H = case["halo"]
    rx0 = receiver_for(case, keep=False, max_samples=n)
    d0 = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
    rx0.process(case["codes"].cuda(), case["first"], n, ref=case["ref"].cuda(), decisions=d0)
    rx1 = receiver_for(case, keep=False, max_samples=chunk)
    d1 = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
    ref = case["ref"].cuda()
    first = case["first"]

    def process(w, f0, nc):
        o = (f0 - first) // 4
        rx1.process(w, f0, nc, ref=ref[o:o + nc // 4], decisions=d1[o:o + nc // 4])

    sh = shard.plan_weak(n, 1, stream_first=first, halo=H)
    host = case["codes"].pin_memory()
    got = ingest.distribute(sh, chunk, process, host_stream=host, stream_first=first - H,
                            device=torch.device("cuda"))
    torch.cuda.synchronize()
    assert got == n + 3 * 2 * H
    assert torch.equal(d0, d1)
    assert rx0.stats() == rx1.stats()
    rx0.close()
    rx1.close()
