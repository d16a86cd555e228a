"""Fig. 2b / 2c analogues through the B200 receiver on the nonlinear channel workload
(kkgen/ssfm.py): Q vs launch power at each format's limit distance, and the optimum
launch power vs distance for 4- and 32-QAM. Each point: one periodic 2,048,000-sample block (125 frames)
propagated on the GPU (single channel SSFM + ASE), received with kk_process_frames (block-LS + CPR), Q from
the BER (ties at zero errors broken by the decision-directed EVM SNR); CSPR optimised over a small grid as
in the paper ("launch power ... and its CSPR were optimized").

  python tools/ssfm_sweep.py --out profiles/r01_ssfm_fig2.json
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
from paper_2104_06311_b200 import KK_STAGE_EQ, Receiver, kkrx  # noqa: E402

LIMITS = {4: 100, 8: 76, 16: 56, 32: 36, 64: 16}   # spans: PAPER.md:106 limit distances (10000 … 1600 km)


def q_point(M, spans, p_dbm, cspr, dev, seed=7):
    cfg = kkgen.LinkConfig(formats=(M,), cspr_db=cspr, seed=seed + M)
    halo = 16640
    w = ssfm.workload(cfg, ssfm.FiberLink(), ssfm.BLOCK, p_dbm, halo, n_spans=spans, device=dev)
    rx = Receiver(adc_scale=w["adc_scale"], ref_intensity=w["i_ref"], dispersion_ps_per_nm=w["dl_ps_nm"],
                  formats=(M,), max_samples_per_call=ssfm.BLOCK, keep_intermediate=True)
    dec = torch.empty(ssfm.BLOCK // 4, dtype=torch.uint8, device=dev)
    rx.process(w["codes"], 0, ssfm.BLOCK, ref=w["labels"].contiguous(), decisions=dec)
    z = rx.intermediate(KK_STAGE_EQ)[1].to(torch.complex128)
    st = rx.stats()
    rx.close()
    pts = torch.from_numpy(kkgen.tx_alphabet(M)).to(dev)[dec.to(torch.int64)]
    snr = 10 * math.log10(float(torch.mean(torch.abs(pts) ** 2) / torch.mean(torch.abs(z - pts) ** 2)))
    bits, be = sum(st["bits"]), sum(st["bit_err"])
    ber = be / bits
    q = kkrx.kk_q_from_ber(ber) if 0 < ber < 0.5 else (None if ber >= 0.5 else float("inf"))
    return dict(M=M, spans=spans, km=spans * 100, p_dbm=p_dbm, cspr_db=cspr, ber=ber, q_db=q,
                snr_evm_db=snr, osnr_db=w["osnr_db"], bad_frames=st["bad_frames"])


def _key(d):   # lower BER first; ties (e.g. no errors) broken by the decision-directed EVM SNR
    return (d["ber"], -d["snr_evm_db"])


def best_over_cspr(M, spans, p, csprs, dev):
    pts = [q_point(M, spans, p, c, dev) for c in csprs]
    return min(pts, key=_key), pts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--powers", type=float, nargs="+", default=[-16, -14, -12, -10, -8, -6, -4, -2, 0])
    ap.add_argument("--csprs", type=float, nargs="+", default=[6.0, 8.0, 10.0])
    ap.add_argument("--out", default="")
    ap.add_argument("--fig", default="2bc", choices=["2bc", "2a"])
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    t0 = time.time()
    if a.fig == "2a":
        # Q vs distance per format, launch power and CSPR optimised per point ("For each point, the
        # launch power of the test channel ... and its CSPR were optimized")
        dist = {4: (20, 40, 60, 80, 100), 8: (16, 36, 56, 76, 96), 16: (16, 28, 40, 56, 72), 32: (8, 16, 24, 36, 48),
                64: (4, 8, 12, 16, 24)}
        fig2a = []
        for M, spans_list in dist.items():
            for spans in spans_list:
                pts = [best_over_cspr(M, spans, p, a.csprs, dev)[0] for p in a.powers]
                opt = min(pts, key=_key)
                fig2a.append(dict(M=M, km=spans * 100, p_opt_dbm=opt["p_dbm"], cspr_db=opt["cspr_db"],
                                  q_db=opt["q_db"], ber=opt["ber"], snr_evm_db=opt["snr_evm_db"]))
                print("2a", fig2a[-1], flush=True)
        if a.out:
            json.dump(dict(fig2a=fig2a, block_samples=ssfm.BLOCK, link=vars(ssfm.FiberLink()),
                           seconds=time.time() - t0), open(a.out, "w"), indent=1)
        return
    fig2b = []
    for M, spans in LIMITS.items():
        for p in a.powers:
            best, _ = best_over_cspr(M, spans, p, a.csprs, dev)
            fig2b.append(best)
            print("2b", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in best.items()}, flush=True)
    fig2c = []
    for M, dist in ((4, (20, 40, 60, 80, 100)), (32, (8, 16, 24, 36))):
        for spans in dist:
            pts = [best_over_cspr(M, spans, p, a.csprs, dev)[0] for p in a.powers]
            opt = min(pts, key=_key)
            fig2c.append(dict(M=M, km=spans * 100, p_opt_dbm=opt["p_dbm"], q_db=opt["q_db"], ber=opt["ber"],
                              snr_evm_db=opt["snr_evm_db"], cspr_db=opt["cspr_db"]))
            print("2c", fig2c[-1], flush=True)
    res = dict(fig2b=fig2b, fig2c=fig2c, block_samples=ssfm.BLOCK, link=vars(ssfm.FiberLink()),
               seconds=time.time() - t0)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
