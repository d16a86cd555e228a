"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times (calls of
min(2^28, S) samples),
checked on frames sampled across the stream (the oracle recomputes each sampled run of frames from the same
int16 codes with its halo), plus properties that hold at any size (counts add up, chunking invariance).

configs (BASELINE.json): C2 16-QAM 5600 km 2^22 (CSPR 6 dB at OSNR 17 dB — clamps occur), C3 64-QAM 1600 km
2^24, C4 4-QAM 10,000 km 2^26 (L = 15), C5 mixed 4→64-QAM 2^32 per GPU (the bench workload).
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import kkgen  # noqa: E402
from oracle import receiver as R  # noqa: E402
from oracle import theory  # noqa: E402
from paper_2104_06311_b200 import Receiver  # noqa: E402

F, H = 16384, 16640
CHUNK = 1 << 29          # bench.py --chunk default


def _run_stream(lc, S, first=0, chunk=CHUNK):
    dev = torch.device("cuda", 0)
    g = kkgen.generate(lc, first - H, first + S + H, device=dev, chunk=1 << 24)
    codes, ref = g["codes"], g["labels"][H // 4:(H + S) // 4]
    rx = Receiver(adc_scale=lc.adc_scale, ref_intensity=lc.i_ref, dispersion_ps_per_nm=lc.dl_ps_nm,
                  formats=lc.formats, segment_frames=lc.segment_frames, max_samples_per_call=min(chunk, S))
    dec = torch.empty(S // 4, dtype=torch.uint8, device=dev)
    c = min(chunk, S)
    for c0 in range(0, S, c):
        rx.process(codes, first + c0, c, ref=ref[c0 // 4:(c0 + c) // 4], decisions=dec[c0 // 4:(c0 + c) // 4],
                   offset=c0)
    st = rx.stats()
    rx.close()
    return codes, ref, dec, st


def _oracle_frames(lc, codes, ref, first, f0, nfr):
    """Oracle on frames [f0, f0 + nfr) (stream-relative) from the same codes."""
    s0 = f0 * F
    c = codes[s0: s0 + nfr * F + 2 * H].cpu().numpy()
    r = ref[s0 // 4:(s0 + nfr * F) // 4].cpu().numpy()
    cfg = R.OracleConfig(dispersion_ps_per_nm=lc.dl_ps_nm, adc_scale=lc.adc_scale, ref_intensity=lc.i_ref,
                         formats=tuple(lc.formats), segment_frames=lc.segment_frames)
    return R.receive(c, first + s0, nfr * F, cfg, ref=r, keep=False)


def _check_sampled(lc, S, picks, nfr=2, first=0, chunk=CHUNK, min_agree=0.9999):
    codes, ref, dec, st = _run_stream(lc, S, first, chunk)
    total_frames = S // F
    assert st["frames"] == total_frames and st["bad_frames"] == 0 and st["dead_frames"] == 0
    assert sum(st["sym"]) == S // 4
    agree = n = 0
    be_g = be_o = 0
    dec_h = dec.cpu().numpy()
    for f0 in picks:
        f0 = min(f0, total_frames - nfr)
        o = _oracle_frames(lc, codes, ref, first, f0, nfr)
        d = dec_h[f0 * 4096:(f0 + nfr) * 4096]
        agree += int(np.sum(d == o["dec"]))
        n += len(d)
        r = ref[f0 * 4096:(f0 + nfr) * 4096].cpu().numpy().astype(np.int64)
        be_g += int(np.sum([bin(x).count("1") for x in (d.astype(np.int64) ^ r)]))
        be_o += int(o["counts"]["bit_err"].sum())
    assert agree / n >= min_agree, (agree, n)
    return st, be_g, be_o, n


def test_c2_full_size():
    lc = kkgen.WORKLOADS["C2"]["cfg"]
    st, bg, bo, n = _check_sampled(lc, 1 << 22, picks=[0, 63, 127, 200, 254])
    # the whole 2^22 stream through the oracle too (it finishes in seconds): Q within 0.05 dB
    codes, ref, dec, st2 = _run_stream(lc, 1 << 22)
    o = _oracle_frames(lc, codes, ref, 0, 0, 256)
    bits = sum(st2["bits"])
    qg = theory.q_from_ber(sum(st2["bit_err"]) / bits)
    qo = theory.q_from_ber(int(o["counts"]["bit_err"].sum()) / bits)
    assert abs(qg - qo) <= 0.05, (qg, qo)
    assert st2["clamped"] == o["counts"]["clamped"]
    assert np.mean(dec.cpu().numpy() == o["dec"]) >= 0.9999


def test_c3_full_size_sampled():
    lc = kkgen.WORKLOADS["C3"]["cfg"]
    _check_sampled(lc, 1 << 24, picks=[0, 255, 511, 767, 1022])


def test_c4_full_size_sampled():
    lc = kkgen.WORKLOADS["C4"]["cfg"]
    st, bg, bo, n = _check_sampled(lc, 1 << 26, picks=[0, 1023, 2047, 3071, 4094])
    assert bg > 0 and abs(bg - bo) <= max(3, 0.01 * bo)


def test_c5_bench_shard_sampled():
    """The bench workload exactly: 2^32 samples of the mixed-format stream on one GPU in 2^29-sample calls;
    sampled frames include every format, format switches, both ends of the shard and runs straddling call
    boundaries (32768 frames per call: the pick 2·16384 − 1 straddles the first)."""
    lc = kkgen.WORKLOADS["C5"]["cfg"]
    S = 1 << 32
    nf = S // F
    picks = [0, 255, 256 + 255, 1023 + 128, 1024 + 256 * 3, 16383, 16384 + 255, 2 * 16384 - 1, nf // 2, nf - 2]
    st, bg, bo, n = _check_sampled(lc, S, picks=picks, nfr=2)
    assert all(v > 0 for v in st["sym"])    # every format of the schedule was received
    assert st["bit_err"][4] > 0          # 64-QAM at 26 dB has errors


def test_c5_second_rank_shard_matches_whole_stream():
    """Weak-scaling shard of rank 1 (global samples [2^28, 2^29)) decides exactly like the same frames
    processed inside a longer single-GPU stream (no cross-shard state)."""
    lc = kkgen.WORKLOADS["C5"]["cfg"]
    S = 1 << 28
    _, _, dec1, _ = _run_stream(lc, S, first=S)
    _, _, dec_all, _ = _run_stream(lc, 2 * S, first=0)
    assert torch.equal(dec1, dec_all[S // 4:])


def test_c5_whole_stream_in_one_call_matches_bench_chunking():
    """Maximum call size: the whole 2^32-sample C5 stream in ONE kk_process_frames call (2^18 frames, 2^31 2-sps
    MF outputs — every 64-bit index path, the K3 tensor maps over 2^28 rows) decides and counts exactly like the
    bench's 2^29-sample calls (every grid is anchored at global sample 0)."""
    lc = kkgen.WORKLOADS["C5"]["cfg"]
    S = 1 << 32
    dev = torch.device("cuda", 0)
    g = kkgen.generate(lc, -H, S + H, device=dev, chunk=1 << 24)
    codes, ref = g["codes"], g["labels"][H // 4:(H + S) // 4]
    del g
    outs = []
    for chunk in (S, CHUNK):
        rx = Receiver(adc_scale=lc.adc_scale, ref_intensity=lc.i_ref, dispersion_ps_per_nm=lc.dl_ps_nm,
                      formats=lc.formats, segment_frames=lc.segment_frames, max_samples_per_call=chunk)
        dec = torch.empty(S // 4, dtype=torch.uint8, device=dev)
        for c0 in range(0, S, chunk):
            rx.process(codes, c0, chunk, ref=ref[c0 // 4:(c0 + chunk) // 4], decisions=dec[c0 // 4:(c0 + chunk) // 4],
                       offset=c0)
        outs.append((dec, rx.stats()))
        rx.close()
        torch.cuda.empty_cache()
    (d1, s1), (d2, s2) = outs
    assert s1 == s2, (s1, s2)
    assert s1["frames"] == S // F and sum(s1["sym"]) == S // 4
    assert torch.equal(d1, d2)
