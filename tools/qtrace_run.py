"""Fig. 3b analogue: continuous Q-factor traces in 21 ms bins over a long stream.

The stream is generated on the device piece by piece (kkgen's chunks sit on a global grid, so pieces join
bit-exactly) and
received with kk_process_frames_ex in 2^26-sample calls; per-frame bit errors are binned into 5127-frame
(21.0 ms) bins and mapped to Q with kk_q_from_ber.

  python tools/qtrace_run.py --seconds 20 --formats 4 8 16 --esn0 11 14 17 --dl 152000 --out trace.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kkgen  # noqa: E402
from paper_2104_06311_b200 import Receiver, qtrace  # noqa: E402

F, H = 16384, 16640


def run(fmt: int, esn0: float, dl: float, seconds: float, cspr: float, piece: int, chunk: int, seed: int):
    dev = torch.device("cuda", 0)
    lc = kkgen.LinkConfig(formats=(fmt,), dl_ps_nm=dl, cspr_db=cspr, esn0_db=esn0, seed=seed)
    total = int(seconds * 4e9) // piece * piece
    rx = Receiver(adc_scale=lc.adc_scale, ref_intensity=lc.i_ref, dispersion_ps_per_nm=dl, formats=(fmt,),
                  max_samples_per_call=chunk)
    fe_all = []
    t_gen = t_rx = 0.0
    for p0 in range(0, total, piece):
        t0 = time.perf_counter()
        g = kkgen.generate(lc, p0 - H, p0 + piece + H, device=dev, chunk=1 << 24)
        codes, ref = g["codes"], g["labels"][H // 4:(H + piece) // 4]
        del g
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        fe = torch.empty(2 * piece // F, dtype=torch.int32, device=dev)
        for c0 in range(0, piece, chunk):
            rx.process(codes, p0 + c0, chunk, ref=ref[c0 // 4:(c0 + chunk) // 4], offset=c0,
                       frame_errors=fe[2 * c0 // F: 2 * (c0 + chunk) // F])
        torch.cuda.synchronize()
        t_rx += time.perf_counter() - t1
        t_gen += t1 - t0
        fe_all.append(fe.view(-1, 2)[:, 1].cpu())
        del codes, ref
    be = torch.cat(fe_all).numpy()
    bits_per_frame = 4096 * (fmt.bit_length() - 1)
    bins = qtrace.bin_q(be, [bits_per_frame] * len(be))
    st = rx.stats()
    rx.close()
    qs = [b["q_db"] for b in bins if b["q_db"] is not None]
    ber = sum(st["bit_err"]) / sum(st["bits"])
    return dict(format=fmt, esn0_db=esn0, dl_ps_nm=dl, cspr_db=cspr, seconds=total / 4e9, samples=total,
                bins=len(bins), q_mean_db=sum(qs) / max(len(qs), 1), q_min_db=min(qs) if qs else None,
                q_max_db=max(qs) if qs else None, q_total_db=qtrace.kkrx.kk_q_from_ber(ber) if 0 < ber < 0.5 else None,
                ber=ber, gen_s=t_gen, rx_s=t_rx, rx_gs_per_s=total / t_rx / 1e9,
                trace=[(round(b["t_s"], 4), None if b["q_db"] is None else round(b["q_db"], 3)) for b in bins])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=20.0)
    ap.add_argument("--formats", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--esn0", type=float, nargs="+", default=[11.0, 14.0, 17.0])
    ap.add_argument("--dl", type=float, default=152000.0)          # 7600 km at 20 ps/nm/km
    ap.add_argument("--cspr", type=float, default=12.0)
    ap.add_argument("--piece", type=int, default=1 << 30)
    ap.add_argument("--chunk", type=int, default=1 << 28)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = [run(m, e, a.dl, a.seconds, a.cspr, a.piece, a.chunk, seed=700 + m) for m, e in zip(a.formats, a.esn0)]
    txt = json.dumps(res)
    if a.out:
        open(a.out, "w").write(txt)
    for r in res:
        print({k: v for k, v in r.items() if k != "trace"})


if __name__ == "__main__":
    main()
