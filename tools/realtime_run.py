"""Sustained real-time run through host ingest (§3: "continuous real-time performance ... during 20
second periods ... Q-factors were estimated from BER in bins of 21 ms"; VERDICT r01 "What's missing" 3).

A periodic receiver input is generated once on the GPU with the nonlinear channel workload (kkgen/ssfm.py: a
periodic launch field of P samples, split-step fibre propagation with EDFA ASE, square law, int16 ADC — the period
is a multiple of BLOCK = lcm(16384, 1000), so frames and the 0.516 GHz tone phase repeat exactly) and copied to
pinned HOST memory, tiled so that any call of the stream finds its window (core + halos) and its labels at host
offset (first mod P). The stream is then received for `--seconds` of signal through the library's end-to-end call
kk_process_frames_host (host→device copies, two staging streams, decisions copied back) in calls of one 21 ms bin
each (5127 frames); after each call kk_stats gives the bin's error counts. Reported per bin: Q (from the bin's BER),
the wall time of the call and the real-time margin (signal duration / wall time, > 1 = faster than real time).

  python tools/realtime_run.py --seconds 20 --out profiles/r02_realtime_20s.json
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kkgen  # noqa: E402
from kkgen import ssfm  # noqa: E402
from paper_2104_06311_b200 import Receiver, kkrx  # noqa: E402

F = 16384
BIN_FRAMES = 5127                      # 5127 × 4096 symbols at 1 GBaud = 21.0 ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=20.0)
    ap.add_argument("--format", type=int, default=16)
    ap.add_argument("--spans", type=int, default=20, help="100-km spans (20 → 2000 km)")
    ap.add_argument("--power-dbm", type=float, default=-2.0)
    ap.add_argument("--cspr", type=float, default=8.0)
    ap.add_argument("--period-blocks", type=int, default=16, help="period P = this × 2,048,000 samples")
    ap.add_argument("--adc-bits", type=int, default=15)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)

    # ---- one periodic period of the receiver input (GPU), then pinned host copies tiled for any call offset
    P = a.period_blocks * ssfm.BLOCK
    L = BIN_FRAMES * F                                        # samples per call = one bin
    cfg = kkgen.LinkConfig(formats=(a.format,), cspr_db=a.cspr, seed=800 + a.format, adc_bits=a.adc_bits)
    link = ssfm.FiberLink()
    t0 = time.perf_counter()
    w = ssfm.workload(cfg, link, P, a.power_dbm, 0, n_spans=a.spans, device=dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    block, labels = w["codes"], w["labels"].to(torch.uint8)
    rx = Receiver(adc_scale=w["adc_scale"], ref_intensity=w["i_ref"], dispersion_ps_per_nm=w["dl_ps_nm"],
                  formats=(a.format,), max_samples_per_call=1 << 26, device=0, input_uint8=a.adc_bits <= 8)
    H = rx.halo
    reps = (P + L + 2 * H) // P + 2
    idx = torch.remainder(torch.arange(-H, P + L + H, device=dev), P)
    h_codes = torch.empty(P + L + 2 * H, dtype=block.dtype, pin_memory=True)
    h_codes.copy_(block[idx])
    lidx = torch.remainder(torch.arange(0, (P + L) // 4, device=dev), P // 4)
    h_ref = torch.empty((P + L) // 4, dtype=torch.uint8, pin_memory=True)
    h_ref.copy_(labels[lidx])
    h_dec = torch.empty(L // 4, dtype=torch.uint8, pin_memory=True)
    del idx, lidx, reps

    # ---- the stream: n_bins calls of one bin each, global samples [b·L, (b+1)·L)
    n_bins = int(math.ceil(a.seconds * 4e9 / L))
    bits_bin = L // 4 * int(round(math.log2(a.format)))
    rx.process_host(h_codes, 0, L, ref=h_ref, decisions=h_dec)          # warm-up (staging allocations)
    rx.reset_stats()
    prev = rx.stats()
    bins = []
    t_all = time.perf_counter()
    for b in range(n_bins):
        first = b * L
        off = first % P                                                 # host offset of this call's window
        t1 = time.perf_counter()
        rx.process_host(h_codes, first, L, ref=h_ref[off // 4:], decisions=h_dec, offset=off)
        st = rx.stats()                                                 # D2H of the bin's counters
        dt = time.perf_counter() - t1
        be = sum(st["bit_err"]) - sum(prev["bit_err"])
        se = sum(st["sym_err"]) - sum(prev["sym_err"])
        prev = st
        ber = be / bits_bin
        bins.append(dict(t_s=round(first / 4e9, 5), bit_err=be, sym_err=se,
                         q_db=(kkrx.kk_q_from_ber(ber) if 0 < ber < 0.5 else None), wall_ms=round(dt * 1e3, 3),
                         margin=round((L / 4e9) / dt, 3)))
    wall = time.perf_counter() - t_all
    rx.close()
    qs = [x["q_db"] for x in bins if x["q_db"] is not None]
    margins = [x["margin"] for x in bins]
    tot_be = sum(x["bit_err"] for x in bins)
    out = dict(
        what="sustained real-time reception through kk_process_frames_host (pinned host buffers, H2D copies, "
             "decisions D2H) of a periodic SSFM-channel stream; one call per 21 ms bin",
        format=a.format, spans=a.spans, dl_ps_nm=w["dl_ps_nm"], osnr_db=w["osnr_db"], power_dbm=a.power_dbm,
        cspr_db=a.cspr, adc_bits=a.adc_bits, period_samples=P, bin_samples=L, bins=n_bins,
        signal_seconds=n_bins * L / 4e9, wall_seconds=wall, gen_seconds=t_gen,
        sustained_gs_per_s=n_bins * L / wall / 1e9, real_time_factor=(n_bins * L / 4e9) / wall,
        margin_min=min(margins), margin_median=sorted(margins)[len(margins) // 2],
        bins_below_real_time=sum(1 for m in margins if m < 1.0),
        q_total_db=(kkrx.kk_q_from_ber(tot_be / (bits_bin * n_bins)) if tot_be else None),
        q_bin_min_db=min(qs) if qs else None, q_bin_max_db=max(qs) if qs else None,
        h2d_bytes_per_bin=(L + 2 * H) * h_codes.element_size() + L // 4, d2h_bytes_per_bin=L // 4 + 192,
        trace=bins)
    txt = json.dumps(out)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt)
    print(json.dumps({k: v for k, v in out.items() if k != "trace"}))


if __name__ == "__main__":
    main()
