"""Nonlinear fiber channel workload (SPEC S:203–248 channel module) — input generation.

Like the rest of `kkgen`, this builds the receiver's INPUT (int16 ADC codes + transmitted labels) and holds
none of the receiver's arithmetic. It propagates the paper's minimum-phase test signal through the paper's
link (100 × ~100 km spans of submarine fibre, 0.154 dB/km, A_eff 112 µm², EDFAs) with the
scalar nonlinear Schrödinger equation, single channel (SPM; WDM dummy channels are not simulated, SPEC's
design ledger), so the Fig. 2b/2c trends (Q vs launch power with an interior optimum, optimum power falling
with distance) can be produced through the same B200 receiver (`tools/ssfm_sweep.py`).

Model (all fp64 torch, CPU or CUDA):
  * transmitter: one periodic block of N samples at 8 GS/s (2× the ADC rate): symbols from kkgen's labels
    (same hash, same alphabets), RRC 1 % by its exact frequency response, data shifted to +0.516 GHz by an
    integer number of FFT bins (residual offset ≤ 8 GHz / 2N), tone A at DC with A² = CSPR·P_x, total
    power = the launch power P_ch;
  * per span (length L, α, β₂ = −Dλ²/(2πc), γ = 2π·n₂/(λ·A_eff)): symmetric split step with `steps`
    equal steps — ½ linear (exp(+iβ₂ω²h/2 − αh/2) on the spectrum) / nonlinear exp(+iγ|E|²·L_eff) with
    L_eff = 2·sinh(αh/2)/α (exact for the midpoint power) /
    ½ linear; then an EDFA restoring the span loss exactly and adding circular complex ASE of PSD
    n_sp·hν·(G − 1), n_sp = NF/2 (single polarisation), drawn from kkgen's counter-based Gaussian keyed by
    (seed, span, sample);
  * receiver front end: |E|² at 8 GS/s, ideal low-pass to ±2 GHz and decimation to 4 GS/s, int16 ADC with
    full scale 1.1·max(I); the block repeats periodically, so the receiver's halos wrap around.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import BAUD, C_LIGHT, F_C, FS, LAMBDA_M, ROLLOFF, LinkConfig, gauss_complex, symbol_labels, tx_alphabet

H_PLANCK = 6.62607015e-34
UP = 2                      # simulation rate = UP × ADC rate
FS_SIM = UP * FS


@dataclass
class FiberLink:
    span_km: float = 100.0                # PAPER.md:50 "average span length was approximately 100 km"
    n_spans: int = 100                    # PAPER.md:50 "100 span straight-line link"
    alpha_db_km: float = 0.154
    d_ps_nm_km: float = 20.0              # SURVEY §8 (D ≈ 20 ps/nm/km class submarine fibre)
    aeff_um2: float = 112.0
    n2_m2_w: float = 2.6e-20              # SPEC design ledger
    nf_db: float = 5.0                    # EDFA noise figure (not given by the paper)
    steps: int = 20                       # split steps per span
    nonlinear: bool = True
    ase: bool = True

    @property
    def alpha_per_m(self) -> float:       # power attenuation coefficient (1/m)
        return self.alpha_db_km / (10.0 * math.log10(math.e)) / 1e3

    @property
    def beta2(self) -> float:             # s²/m
        d = self.d_ps_nm_km * 1e-12 / (1e-9 * 1e3)          # s/m²
        return -d * LAMBDA_M ** 2 / (2 * math.pi * C_LIGHT)

    @property
    def gamma(self) -> float:             # 1/(W·m)
        return 2 * math.pi * self.n2_m2_w / (LAMBDA_M * self.aeff_um2 * 1e-12)

    @property
    def span_gain(self) -> float:         # linear power gain restoring one span
        return 10.0 ** (self.alpha_db_km * self.span_km / 10.0)

    @property
    def ase_psd(self) -> float:           # W/Hz per amplifier, single polarisation
        nu = C_LIGHT / LAMBDA_M
        return 0.5 * 10.0 ** (self.nf_db / 10.0) * H_PLANCK * nu * (self.span_gain - 1.0)

    def dl_ps_nm(self, n_spans: int | None = None) -> float:
        return self.d_ps_nm_km * self.span_km * (self.n_spans if n_spans is None else n_spans)

    def osnr_db(self, p_ch_w: float, n_spans: int | None = None) -> float:
        """OSNR in 0.1 nm (12.5 GHz), single polarisation, ASE only."""
        ns = self.n_spans if n_spans is None else n_spans
        return 10 * math.log10(p_ch_w / (ns * self.ase_psd * 12.5e9))


def _freqs(n: int, device) -> torch.Tensor:
    return torch.fft.fftfreq(n, d=1.0 / FS_SIM, device=device).to(torch.float64)


def rrc_response(f: torch.Tensor, rolloff: float = ROLLOFF, baud: float = BAUD) -> torch.Tensor:
    """Root-raised-cosine amplitude response (peak 1) at frequencies f."""
    af = f.abs()
    f1, f2 = (1 - rolloff) * baud / 2, (1 + rolloff) * baud / 2
    mid = torch.sqrt(0.5 * (1 + torch.cos(math.pi / (rolloff * baud) * (af - f1))))
    return torch.where(af <= f1, torch.ones_like(af), torch.where(af <= f2, mid, torch.zeros_like(af)))


BLOCK = 2048000   # lcm(16384, 1000): whole frames AND an exact 0.516 GHz tone offset (129/2000 of 8 GS/s)


def launch_field(cfg: LinkConfig, n: int, p_ch_w: float, device="cpu", exact: bool = True):
    """Periodic launch field at 8 GS/s for ADC samples [0, n) (n a multiple of 4) and its labels.
    Power: mean |E|² = p_ch_w (W); CSPR from cfg. exact: require the data offset to be an integer number of
    bins (n a multiple of 1000), else the receiver sees a residual carrier offset of up to 4 GHz/n."""
    device = torch.device(device)
    ns = n * UP
    if exact:
        assert (ns * 129) % 2000 == 0, "n must be a multiple of 1000 for an exact 0.516 GHz offset (see BLOCK)"
    nsym = n // 4
    k = torch.arange(nsym, dtype=torch.int64, device=device)
    lab = symbol_labels(cfg, k)
    M = cfg.format_of_symbols(k)
    sym = torch.zeros(nsym, dtype=torch.complex128, device=device)
    for m in sorted(set(int(x) for x in cfg.formats)):
        tab = torch.from_numpy(tx_alphabet(m)).to(device)
        sel = M == m
        sym[sel] = tab[lab[sel].to(torch.int64)]
    u = torch.zeros(ns, dtype=torch.complex128, device=device)
    u[::4 * UP] = sym
    U = torch.fft.fft(u) * rrc_response(_freqs(ns, device))
    shift = int(round(F_C / FS_SIM * ns)) * cfg.sideband            # data to ±0.516 GHz (integer bins)
    x = torch.fft.ifft(torch.roll(U, shift))
    x = x / torch.sqrt(torch.mean(x.real ** 2 + x.imag ** 2))         # P_x = 1 (normalised)
    A = math.sqrt(10.0 ** (cfg.cspr_db / 10.0))
    E = (A + x) * math.sqrt(p_ch_w / (A * A + 1.0))
    return E, lab


def linear_step(E: torch.Tensor, link: FiberLink, h_m: float, w2: torch.Tensor) -> torch.Tensor:
    """CD + loss over h metres: spectrum × exp(+iβ₂ω²h/2 − αh/2)."""
    op = torch.exp(1j * (link.beta2 / 2.0) * w2 * h_m - link.alpha_per_m * h_m / 2.0)
    return torch.fft.ifft(torch.fft.fft(E) * op)


def propagate(E: torch.Tensor, link: FiberLink, seed: int = 0, n_spans: int | None = None) -> torch.Tensor:
    """Symmetric split-step over the spans, EDFA (exact loss inversion) + ASE after each span."""
    ns = E.numel()
    w = 2 * math.pi * _freqs(ns, E.device)
    w2 = w * w
    spans = link.n_spans if n_spans is None else n_spans
    h = link.span_km * 1e3 / link.steps
    a = link.alpha_per_m
    # nonlinear step at the step's midpoint (after ½ step of loss): ∫ P dz over the step = P_mid·2sinh(αh/2)/α
    leff = 2.0 * math.sinh(a * h / 2.0) / a if a > 0 else h
    half = torch.exp(1j * (link.beta2 / 2.0) * w2 * (h / 2) - a * (h / 2) / 2.0)
    full = half * half
    g_amp = math.sqrt(link.span_gain)
    idx = torch.arange(ns, dtype=torch.int64, device=E.device)
    sig_ase = math.sqrt(link.ase_psd * FS_SIM)                         # per-sample complex std (E|n|² = PSD·fs)
    for s in range(spans):
        X = torch.fft.fft(E) * half
        for st in range(link.steps):
            E = torch.fft.ifft(X)
            if link.nonlinear:
                E = E * torch.exp(1j * link.gamma * (E.real ** 2 + E.imag ** 2) * leff)
            X = torch.fft.fft(E) * (full if st < link.steps - 1 else half)
        E = torch.fft.ifft(X) * g_amp
        if link.ase:
            E = E + sig_ase * gauss_complex(seed * 7919 + s, idx)
    return E


def detect(E: torch.Tensor, adc_bits: int = 15):
    """|E|² at 8 GS/s → ideal low-pass ±2 GHz → every other sample → int16 ADC (full scale 1.1·max I).
    Returns codes (periodic block of n = E.numel()/2 samples), adc_scale, mean intensity."""
    I8 = E.real ** 2 + E.imag ** 2
    ns = I8.numel()
    S = torch.fft.fft(I8)
    S[torch.abs(_freqs(ns, E.device)) >= FS / 2] = 0
    I = torch.fft.ifft(S).real[::UP]
    adc_max = (1 << adc_bits) - 1
    i_clip = 1.1 * float(I.max())
    codes = torch.clamp(torch.round(I * (adc_max / i_clip)), 0, adc_max)
    codes = codes.to(torch.uint8 if adc_bits <= 8 else torch.int16)
    return codes, i_clip / adc_max, float(I.mean())


def workload(cfg: LinkConfig, link: FiberLink, n: int, p_ch_dbm: float, halo: int, n_spans: int | None = None,
             device="cpu") -> dict:
    """Receiver input for ADC samples [0, n): codes of [−halo, n + halo) (periodic wrap) + labels [0, n/4)."""
    assert n % 16384 == 0 and n % 1000 == 0, "whole frames and an exact tone offset: n a multiple of BLOCK"
    p = 1e-3 * 10.0 ** (p_ch_dbm / 10.0)
    E, lab = launch_field(cfg, n, p, device)
    E = propagate(E, link, seed=cfg.seed, n_spans=n_spans)
    codes, adc_scale, i_ref = detect(E, cfg.adc_bits)
    idx = torch.remainder(torch.arange(-halo, n + halo, device=codes.device), n)
    ns = link.n_spans if n_spans is None else n_spans
    return dict(codes=codes[idx], labels=lab, adc_scale=adc_scale, i_ref=i_ref, dl_ps_nm=link.dl_ps_nm(ns),
                osnr_db=link.osnr_db(p, ns) if link.ase else None, p_ch_dbm=p_ch_dbm, n_spans=ns)
