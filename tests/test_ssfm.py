"""Pins of the nonlinear channel workload (kkgen/ssfm.py) against SPEC S:203–248's
examples and closed forms. Input generation, not the receiver: these tests keep the channel honest."""
import math

import numpy as np
import torch

import kkgen
from kkgen import ssfm


def _link(**kw):
    base = dict(n_spans=1, nonlinear=False, ase=False)
    base.update(kw)
    return ssfm.FiberLink(**base)


def test_lossless_linear_identity():
    """Noise off, γ = 0, D = 0: loss then exactly compensating gain → output = input."""
    E, _ = ssfm.launch_field(kkgen.LinkConfig(formats=(16,), cspr_db=8.0, seed=1), 4096, 1e-3, exact=False)
    out = ssfm.propagate(E, _link(d_ps_nm_km=0.0, n_spans=3))
    assert torch.max(torch.abs(out - E)) / torch.max(torch.abs(E)) < 1e-12


def test_span_loss_15_4_db():
    """100 km at 0.154 dB/km → power drops by 15.4 dB."""
    link = _link(d_ps_nm_km=0.0)
    E = torch.full((1024,), 1.0 + 0j, dtype=torch.complex128)
    w2 = torch.zeros(1024, dtype=torch.float64)
    out = ssfm.linear_step(E, link, 100e3, w2)
    drop = -10 * math.log10(float(torch.mean(torch.abs(out) ** 2)))
    assert abs(drop - 15.4) < 0.01


def test_constant_envelope_spm_rotation():
    """Constant envelope, CD off, nonlinearity on → pure phase rotation γ·P·L_eff per span, amplitude kept
    (L_eff = (1 − e^{−αL})/α)."""
    link = _link(d_ps_nm_km=0.0, nonlinear=True, n_spans=4, steps=7)
    P = 2e-3
    E = torch.full((256,), math.sqrt(P) + 0j, dtype=torch.complex128)
    out = ssfm.propagate(E, link)
    a, L = link.alpha_per_m, link.span_km * 1e3
    phi = 4 * link.gamma * P * (1 - math.exp(-a * L)) / a
    assert torch.max(torch.abs(torch.abs(out) - math.sqrt(P))) < 1e-6 * math.sqrt(P)
    assert abs(float(torch.angle(out[0])) - (phi - 2 * math.pi * round(phi / (2 * math.pi)))) < 1e-9


def test_linear_link_equals_cd_all_pass():
    """10,000 km noiseless linear = the all-pass exp(+iβ₂ω²L/2) of the accumulated dispersion."""
    E, _ = ssfm.launch_field(kkgen.LinkConfig(formats=(4,), cspr_db=10.0, seed=2), 8192, 1e-3, exact=False)
    link = _link(n_spans=100, steps=3)
    out = ssfm.propagate(E, link)
    w = 2 * math.pi * torch.fft.fftfreq(E.numel(), d=1.0 / ssfm.FS_SIM).to(torch.float64)
    bl = kkgen.beta2_l(link.dl_ps_nm())
    ref = torch.fft.ifft(torch.fft.fft(E) * torch.exp(1j * bl / 2 * w * w))
    assert float(torch.linalg.norm(out - ref) / torch.linalg.norm(ref)) < 1e-9
    assert abs(bl - link.beta2 * 100 * link.span_km * 1e3) < 1e-9 * abs(bl)


def test_ase_accumulates_linearly():
    """ASE noise power after N spans = N × one span's (gain = loss, so each span's ASE arrives intact);
    OSNR falls by 10·log10(N)."""
    link = _link(ase=True, n_spans=8)
    z = torch.zeros(1 << 16, dtype=torch.complex128)
    p1 = float(torch.mean(torch.abs(ssfm.propagate(z, link, seed=3, n_spans=1)) ** 2))
    p8 = float(torch.mean(torch.abs(ssfm.propagate(z, link, seed=3, n_spans=8)) ** 2))
    assert abs(p1 / (link.ase_psd * ssfm.FS_SIM) - 1) < 0.02
    assert abs(10 * math.log10(p8 / p1) - 10 * math.log10(8)) < 0.1
    assert abs(link.osnr_db(1e-3, 1) - link.osnr_db(1e-3, 8) - 10 * math.log10(8)) < 1e-12


def test_step_halving_converges():
    """Halving the split step changes the output by < 1e-3 RMS at a high launch power."""
    cfg = kkgen.LinkConfig(formats=(16,), cspr_db=8.0, seed=4)
    E, _ = ssfm.launch_field(cfg, 8192, 10 ** 0.6 * 1e-3, exact=False)      # +6 dBm
    a = ssfm.propagate(E, _link(nonlinear=True, n_spans=10, steps=20))
    b = ssfm.propagate(E, _link(nonlinear=True, n_spans=10, steps=40))
    assert float(torch.linalg.norm(a - b) / torch.linalg.norm(b)) < 1e-3


def test_exact_tone_offset_block():
    """The data sits exactly at +0.516 GHz only when 2n·129/2000 is an integer (BLOCK = lcm(16384, 1000));
    the launch spectrum then has its data band centred on that bin."""
    n = 4000
    E, _ = ssfm.launch_field(kkgen.LinkConfig(formats=(4,), cspr_db=10.0, seed=6), n, 1e-3)
    S = torch.abs(torch.fft.fft(E - E.mean())) ** 2
    f = torch.fft.fftfreq(2 * n, d=1.0 / ssfm.FS_SIM)
    centroid = float((S * f).sum() / S.sum())
    assert abs(centroid - kkgen.F_C) < 5e6
    assert ssfm.BLOCK % 16384 == 0 and (2 * ssfm.BLOCK * 129) % 2000 == 0
    try:
        ssfm.launch_field(kkgen.LinkConfig(formats=(4,)), 4096, 1e-3)
        raise AssertionError("inexact offset accepted")
    except AssertionError as e:
        assert "multiple of 1000" in str(e)
