"""Shared helpers for the GPU parity tests: build one seeded case, run the oracle and the CUDA path on the
same int16 codes. (Test infrastructure: imports the oracle, which the product never does.)"""
from __future__ import annotations

import math

import numpy as np
import torch

import kkgen
from oracle import receiver as R

F = 16384
HALO = 16640


def make_case(M=4, dl=0.0, cspr=12.0, esn0=None, n=1 << 16, first=2 * F, seed=7, noise="white", formats=None,
              segment_frames=1 << 30, wander_rad=0.0, sideband=1, **ocfg_kw):
    formats = tuple(formats) if formats else (M,)
    lc = kkgen.LinkConfig(formats=formats, segment_frames=segment_frames, dl_ps_nm=dl, cspr_db=cspr,
                          esn0_db=esn0, seed=seed, noise=noise, wander_rad=wander_rad, sideband=sideband)
    ocfg = R.OracleConfig(dispersion_ps_per_nm=dl, adc_scale=lc.adc_scale, ref_intensity=lc.i_ref,
                          formats=formats, segment_frames=segment_frames, sideband=sideband, **ocfg_kw)
    H = R.halo(ocfg)                      # 16640, or 16656 with upsample = 2 (= kk_halo)
    g = kkgen.generate(lc, first - H, first + n + H)
    ref = g["labels"][H // 4:(H + n) // 4].clone()
    return dict(lc=lc, g=g, ocfg=ocfg, first=first, n=n, ref=ref, codes=g["codes"], formats=formats,
                segment_frames=segment_frames, dl=dl, halo=H)


def run_oracle(case, keep=True):
    return R.receive(case["codes"].numpy(), case["first"], case["n"], case["ocfg"], ref=case["ref"].numpy(),
                     keep=keep)


def receiver_for(case, keep=True, max_samples=None, **kw):
    from paper_2104_06311_b200 import Receiver
    o = case["ocfg"]
    return Receiver(adc_scale=o.adc_scale, ref_intensity=o.ref_intensity, dispersion_ps_per_nm=case["dl"],
                    formats=case["formats"], segment_frames=case["segment_frames"],
                    max_samples_per_call=max_samples or max(case["n"], F), keep_intermediate=keep,
                    eq_taps=o.eq_taps, widely_linear=o.eq_widely_linear, cpr_window=o.cpr_window,
                    eq_mode=o.eq_mode, ddlms_block=o.ddlms_block, ddlms_warmup=o.ddlms_warmup,
                    ddlms_mu_warm=o.ddlms_mu_warm, ddlms_mu=o.ddlms_mu, sideband=o.sideband, upsample=o.upsample,
                    **kw)


def run_gpu(case, keep=True, chunk=None, rx=None):
    """Run the CUDA path over the case's core in calls of `chunk` samples; returns decisions, z (last call
    if chunked: full z only when chunk is None), E/y of the (single) call, stats."""
    from paper_2104_06311_b200 import KK_STAGE_EQ, KK_STAGE_FIELD, KK_STAGE_MF
    first, n = case["first"], case["n"]
    rx = rx or receiver_for(case, keep=keep, max_samples=chunk or n)
    codes = case["codes"].cuda()
    ref = case["ref"].cuda()
    dec = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
    chunk = chunk or n
    zs = []
    for c0 in range(0, n, chunk):
        rx.process(codes, first + c0, chunk, ref=ref[c0 // 4:(c0 + chunk) // 4], decisions=dec[c0 // 4:(c0 + chunk) // 4],
                   offset=c0)
        if keep:
            zs.append(rx.intermediate(KK_STAGE_EQ)[1].cpu())
    out = dict(dec=dec.cpu().numpy().astype(np.int64), stats=rx.stats(), rx=rx)
    if keep:
        out["z"] = torch.cat(zs).numpy().astype(np.complex128)
        e0, E = rx.intermediate(KK_STAGE_FIELD)
        m0, y = rx.intermediate(KK_STAGE_MF)
        out.update(E0=e0, E=E.cpu().numpy().astype(np.complex128), m0=m0, y=y.cpu().numpy().astype(np.complex128))
    return out


def rel(a, b, denom=None):
    d = np.linalg.norm(a - b)
    return d / np.linalg.norm(b if denom is None else denom)


def field_rel_err(gpu, orc):
    """‖E_gpu − E_or‖ / ‖E_or − A_f‖ over the range K1 produced (core ± one frame) — SURVEY §8(c)."""
    assert gpu["E0"] == orc["E0"]
    E_or = orc["E"]
    A = np.repeat(orc["A"], F)
    return rel(gpu["E"], E_or, E_or - A)


def eq_check(z_gpu, z_or, tol=1e-4, flip_tol=2e-3, max_flip_frac=0.25, frame_symbols=4096):
    """Equalizer-output parity per frame (DESIGN.md §3 "EQ tolerance and training-decision flips"): every
    frame whose decision-directed training decisions agree is within `tol` relative RMS (global over those
    frames); a pass-1 decision that fp32 and fp64 take differently at a slicer boundary moves that frame's
    taps by O(|Δd|/N) ≈ 1.5e-4 per flip — such frames (error > tol) must be few (≤ max_flip_frac, at least
    one allowed) and bounded by flip_tol. Returns (clean-frame error, flipped frames, worst frame)."""
    zg = np.asarray(z_gpu).reshape(-1, frame_symbols)
    zo = np.asarray(z_or).reshape(-1, frame_symbols)
    fe = np.linalg.norm(zg - zo, axis=1) / np.maximum(np.linalg.norm(zo, axis=1), 1e-30)
    clean = fe <= tol
    n_flip = int(np.sum(~clean))
    assert n_flip <= max(1, int(max_flip_frac * len(fe))), f"EQ: {n_flip}/{len(fe)} frames over {tol}: {fe}"
    assert fe.max() <= flip_tol, f"EQ worst frame {fe.max():.3e} > {flip_tol}"
    ce = rel(zg[clean], zo[clean]) if clean.any() else 0.0
    assert ce <= tol, f"EQ rel err on clean frames {ce:.3e}"
    return ce, n_flip, float(fe.max())
