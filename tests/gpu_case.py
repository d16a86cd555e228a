"""Shared helpers for the GPU parity tests: build one seeded case, run the oracle and the CUDA path on the
same int16 codes. (Test infrastructure: imports the oracle, which the product never does.)"""
from __future__ import annotations

import math
import os

import numpy as np
import torch

import kkgen
from oracle import receiver as R

F = 16384
HALO = 16640


def make_case(M=4, dl=0.0, cspr=12.0, esn0=None, n=1 << 16, first=2 * F, seed=7, noise="white", formats=None,
              segment_frames=1 << 30, wander_rad=0.0, wander_hz=50e3, linewidth_hz=0.0, sideband=1,
              label_source="hash", **ocfg_kw):
    formats = tuple(formats) if formats else (M,)
    lc = kkgen.LinkConfig(formats=formats, segment_frames=segment_frames, dl_ps_nm=dl, cspr_db=cspr,
                          esn0_db=esn0, seed=seed, noise=noise, wander_rad=wander_rad, wander_hz=wander_hz,
                          linewidth_hz=linewidth_hz, sideband=sideband, label_source=label_source)
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
                    ddlms_mu_warm=o.ddlms_mu_warm, ddlms_mu=o.ddlms_mu, ddlms_mu_mid=o.ddlms_mu_mid,
                    sideband=o.sideband, upsample=o.upsample, static_cd=o.static_cd,
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


def _near_boundary(z, M, delta):
    """Indices of z within `delta` (unit-energy units) of a decision boundary, with the point across it:
    t = (|z − p₂|² − |z − p₁|²) / (2|p₂ − p₁|) is the distance to the bisector of the two nearest points."""
    from oracle import constellation as C
    pts, _ = C.constellation(M)
    d2 = np.abs(np.asarray(z).reshape(-1, 1) - pts[None, :]) ** 2
    o = np.argsort(d2, axis=1)[:, :2]
    r = np.arange(len(d2))
    p1, p2 = pts[o[:, 0]], pts[o[:, 1]]
    t = (d2[r, o[:, 1]] - d2[r, o[:, 0]]) / (2 * np.abs(p2 - p1))
    idx = np.nonzero(t < delta)[0]
    return [(int(k), p2[k], float(t[k])) for k in idx]


class _Decide:
    """Hard decision D for the oracle's `decide` hook: brute-force nearest, except that the listed
    (call number, index) pairs take the point across the boundary; records every call's input."""

    def __init__(self, flips=()):
        self.flips = {}
        for c, k, p in flips:
            self.flips.setdefault(c, {})[k] = p
        self.calls = []

    def __call__(self, z, M):
        from oracle import constellation as C
        pts, labs = C.nearest(z, M)
        c = len(self.calls)
        self.calls.append(np.array(z, copy=True))
        if c in self.flips:
            pts = pts.copy()
            allp, alll = C.constellation(M)
            for k, p in self.flips[c].items():
                pts.reshape(-1)[k] = p
                labs.reshape(-1)[k] = alll[np.argmin(np.abs(allp - p))]
        return pts, labs


def _frame_rerun(orc, cfg, fi, flips):
    """z of frame fi recomputed by the oracle with the given decision flips (O8 pass 1 = call 0, O8 unbias =
    call 1, O9 CPR = call 2 of the block-LS path; call i = symbol i of a DDLMS block)."""
    Fs = cfg.frame_symbols
    M = cfg.fmt_of_frame(orc["first"] // cfg.frame_samples + fi)
    K, k0 = orc["K"], fi * Fs
    yf = orc["y"][2 * k0: 2 * k0 + 2 * Fs - 1 + 2 * K]
    dec = _Decide(flips)
    u, _ = R.o8_equalize_frame(yf, K, orc["w_cd"], M, cfg, decide=dec)
    z, _ = R.o9_cpr(u, M, cfg.cpr_window, decide=dec)
    return z, dec, M


def _ddlms_block_rerun(orc, cfg, fi, bb, flips):
    B, W = cfg.ddlms_block, cfg.ddlms_warmup
    kg0 = orc["first"] // cfg.sps + fi * cfg.frame_symbols + bb
    Ms = R._symbol_formats(kg0 - W, W + B, cfg)               # one QAM order per call (= per symbol)
    dec = _Decide(flips)
    z = R.o8_ddlms_block(orc["y"], orc["m0"], kg0 - W, W, B, Ms, cfg, decide=dec)
    return z, dec, Ms


def _prove_flip(target, rerun, tol, delta, max_flips=4):
    """Find decision flips at slicer boundaries (|t| < delta) that make the oracle's recomputed output equal
    `target` within `tol`: greedy over the candidates of the unflipped run (one call at a time). Returns the
    list of flips (proof) or None."""
    z, dec, M = rerun(())
    err = rel(target, z)
    if err <= tol:
        return []
    flips = []
    for _ in range(max_flips):
        best = None
        cands = [(c, k, p) for c, zc in enumerate(dec.calls)
                 for (k, p, _t) in _near_boundary(zc, int(M[c]) if np.ndim(M) else M, delta)
                 if (c, k) not in {(f[0], f[1]) for f in flips}]
        for cand in cands:
            zt, _, _ = rerun(tuple(flips) + (cand,))
            e = rel(target, zt)
            if best is None or e < best[0]:
                best = (e, cand)
        if best is None or best[0] >= err:
            return None
        flips.append(best[1])
        err = best[0]
        if err <= tol:
            return flips
        z, dec, M = rerun(tuple(flips))
    return None


def eq_check(z_gpu, orc, cfg, tol=1e-4, delta=2e-5, frame_symbols=4096):
    """Equalizer-output parity per frame (DESIGN.md §3 "EQ tolerance and training-decision flips").

    Every frame must be within `tol` relative RMS of the oracle — or be PROVEN to differ only by decisions
    that fp32 and fp64 take differently at a slicer boundary: the oracle, re-run on that frame with ≤ 4
    decisions moved across a boundary they sit within `delta` (unit-energy units, ≈ 20× the fp32 error of
    the decided values) of, reproduces the GPU's output within `tol`. Decision points checked: the training
    (pass-1) and unbias decisions of the block LS and the CPR decisions (R10, R12, R27); in DDLMS mode every
    decision of the block's recursion. Returns (error over frames within tol, proven frames, worst raw error)."""
    zg = np.asarray(z_gpu).reshape(-1, frame_symbols)
    zo = np.asarray(orc["z"]).reshape(-1, frame_symbols)
    fe = np.linalg.norm(zg - zo, axis=1) / np.maximum(np.linalg.norm(zo, axis=1), 1e-30)
    clean = fe <= tol
    proven = []
    for fi in np.nonzero(~clean)[0]:
        fi = int(fi)
        if cfg.eq_mode == "ddlms":
            B = cfg.ddlms_block
            for bb in range(0, frame_symbols, B):
                zt = zg[fi, bb:bb + B]
                if rel(zt, zo[fi, bb:bb + B]) <= tol:
                    continue
                proof = _prove_flip(zt, lambda fl: _ddlms_block_rerun(orc, cfg, fi, bb, fl), tol, delta)
                assert proof is not None, f"EQ frame {fi} block {bb}: {rel(zt, zo[fi, bb:bb + B]):.3e} > {tol}, " \
                                          f"no boundary flip explains it"
                proven.append((fi, bb, proof))
        else:
            proof = _prove_flip(zg[fi], lambda fl: _frame_rerun(orc, cfg, fi, fl), tol, delta)
            assert proof is not None, f"EQ frame {fi}: {fe[fi]:.3e} > {tol}, no boundary flip explains it"
            proven.append((fi, proof))
    ce = rel(zg[clean], zo[clean]) if clean.any() else 0.0
    assert ce <= tol, f"EQ rel err on clean frames {ce:.3e}"
    PROOFS.append(dict(test=os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], frames=len(fe),
                       clean_err=float(ce), worst_raw=float(fe.max()),
                       proven=[dict(frame=p[0], block=(p[1] if len(p) == 3 else None),
                                    flips=[dict(call=int(c), index=int(k)) for c, k, _ in p[-1]]) for p in proven]))
    return ce, proven, float(fe.max())


PROOFS = []   # one record per eq_check call (tests/conftest.py writes them to $KK_EQ_PROOF_LOG)


def make_silent_case(M=16, dl=32000.0, n=12 * F, first=2 * F, seed=17, quiet=(2, 9)):
    """Float-intensity input (I/I_ref, so I_ref = 1) whose core frames quiet[0] … quiet[1]−1 carry the tone
    without modulation (I = I_ref exactly): the tone's KK field is exactly constant there, so the frames at
    least two frames inside the quiet stretch have e = E − A_f = 0 and an MF output of exactly zero — no signal
    power to train on (the silent-frame rule: bad frame, z = 0, decisions D(0))."""
    case = make_case(M=M, dl=dl, cspr=12.0, n=n, first=first, seed=seed)
    lc, H = case["lc"], case["halo"]
    I = case["codes"].to(torch.float64) * (lc.adc_scale / lc.i_ref)
    a, b = H + quiet[0] * F, H + quiet[1] * F
    I[a:b] = 1.0
    case["codes"] = I.to(torch.float32)
    case["ocfg"] = R.OracleConfig(dispersion_ps_per_nm=dl, adc_scale=1.0, ref_intensity=1.0, formats=case["formats"])
    case["float_input"] = True
    case["silent_frames"] = list(range(quiet[0] + 2, quiet[1] - 2))
    case["edge_frames"] = [quiet[0] + 1, quiet[1] - 2]   # y partly exactly zero: decided on the oracle's rounding
    return case
