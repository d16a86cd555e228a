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


def test_host_path_orders_after_reset_and_caller_stream():
    """kk_process_frames_host must not race work still queued on the legacy stream (kk_reset_stats
    with stream NULL) or on the caller stream of the context's previous device call — no synchronisation in
    between. Each stream is first kept busy (torch.cuda._sleep) so that an unordered host path would run ahead."""
    from gpu_case import F, make_case, receiver_for
    case = make_case(M=16, dl=112000.0, cspr=10.0, esn0=14.0, n=16 * F, seed=27)
    codes_d, ref_d = case["codes"].cuda(), case["ref"].cuda()
    codes_h, ref_h = case["codes"].pin_memory(), case["ref"].pin_memory()
    rx = receiver_for(case, keep=False, max_samples=4 * F)
    rx.process_host(codes_h, case["first"], case["n"], ref=ref_h)
    want = rx.stats()
    keys = ("sym", "sym_err", "bits", "bit_err", "frames")
    s1 = torch.cuda.Stream()
    for _ in range(3):
        # (a) a device call and the reset queued on a caller stream behind a busy kernel
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            torch.cuda._sleep(50_000_000)
            for c0 in range(0, case["n"], 4 * F):
                rx.process(codes_d, case["first"] + c0, 4 * F, ref=ref_d[c0 // 4:(c0 + 4 * F) // 4], offset=c0,
                           stream=s1)
            rx.reset_stats(stream=s1)
        rx.process_host(codes_h, case["first"], case["n"], ref=ref_h)
        got = rx.stats()
        assert all(got[k] == want[k] for k in keys), ("caller stream", got, want)
        # (b) the reset on the legacy default stream behind a busy kernel
        torch.cuda.synchronize()
        torch.cuda._sleep(50_000_000)                   # current stream = the legacy default stream
        rx.reset_stats()
        rx.process_host(codes_h, case["first"], case["n"], ref=ref_h)
        got = rx.stats()
        assert all(got[k] == want[k] for k in keys), ("legacy stream", got, want)
    rx.close()


def test_device_calls_order_across_caller_streams():
    """Consecutive kk_process_frames / kk_reset_stats / kk_stats_device calls of one context on DIFFERENT caller
    streams, with no synchronisation between them: each waits for the work the previous call queued (they share
    the scratch buffers and the counters). The first stream is kept busy (torch.cuda._sleep) so that an unordered
    call would overtake it: a reset would land before the counts, a second call would overwrite the first's
    scratch mid-flight."""
    from gpu_case import F, make_case, receiver_for
    case = make_case(M=16, dl=112000.0, cspr=10.0, esn0=14.0, n=8 * F, seed=31)
    codes, ref = case["codes"].cuda(), case["ref"].cuda()
    rx = receiver_for(case, keep=False, max_samples=4 * F)
    n, h = case["n"], 4 * F
    want_dec = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
    for c0 in range(0, n, h):                               # reference: one stream, synchronised
        rx.process(codes, case["first"] + c0, h, ref=ref[c0 // 4:(c0 + h) // 4], decisions=want_dec[c0 // 4:(c0 + h) // 4],
                   offset=c0)
    want = rx.stats()
    keys = ("sym", "sym_err", "bits", "bit_err", "frames")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        torch.cuda.synchronize()
        dec = torch.zeros_like(want_dec)
        cnt = torch.zeros(32, dtype=torch.int64, device="cuda")
        with torch.cuda.stream(sa):
            torch.cuda._sleep(50_000_000)
            rx.reset_stats(stream=sa)
            rx.process(codes, case["first"], h, ref=ref[:h // 4], decisions=dec[:h // 4], offset=0, stream=sa)
        # the second half on another stream, then the counters copied on a third (the current) stream
        rx.process(codes, case["first"] + h, h, ref=ref[h // 4:], decisions=dec[h // 4:], offset=h, stream=sb)
        rx.stats_device(cnt)
        torch.cuda.synchronize()
        got = rx.stats()
        assert all(got[k] == want[k] for k in keys), (got, want)
        assert torch.equal(dec, want_dec)
        # the device copy of the counters (words 0–23, kk_stats_t layout) ran after both calls
        assert [int(v) for v in cnt[0:5]] == list(got["sym"]) and int(cnt[21]) == got["frames"]
    rx.close()
