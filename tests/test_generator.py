"""Checks of the shared seeded input generator (kkgen) against the transmitter definitions."""
import math

import numpy as np
import torch

import kkgen


def test_cspr_amplitude_definition():
    # cspr_db = 10 with mean|x|^2 = 0.1 gives A = 1.0 (CSPR = A^2 / P_x)
    assert abs(math.sqrt(0.1 * 10 ** (10 / 10)) - 1.0) < 1e-15
    c = kkgen.LinkConfig(cspr_db=10.0)
    assert abs(c.amp ** 2 / c.px - 10.0) < 1e-12


def test_field_power_cspr_and_single_sidedness():
    cfg = kkgen.LinkConfig(formats=(16,), cspr_db=12.0, seed=5)
    g = kkgen.generate(cfg, 0, 1 << 16, return_field=True)
    E = g["field"].numpy()
    x = E - cfg.amp
    assert abs(np.mean(np.abs(x) ** 2) / cfg.px - 1) < 0.05
    X = np.abs(np.fft.fft(x)) ** 2
    f = np.fft.fftfreq(len(x), d=0.25)              # GHz
    assert np.sum(X[f > 0]) / np.sum(X) > 0.999      # data strictly above the tone (R3)
    band = X[(f > 0.011) & (f < 1.021)].sum() / X.sum()
    assert band > 0.999
    # Parseval on the detected intensity: mean(I) = mean|E|^2
    I = np.abs(E) ** 2
    assert abs(np.mean(I) - np.mean(np.abs(np.fft.fft(E)) ** 2) / len(E)) < 1e-9


def test_chunk_invariance():
    cfg = kkgen.LinkConfig(formats=(4, 16), segment_frames=1, cspr_db=12.0, esn0_db=20.0,
                           dl_ps_nm=200000.0, seed=9)
    a = kkgen.generate(cfg, -4096, 1 << 17, chunk=1 << 20)
    b = kkgen.generate(cfg, -4096, 1 << 17, chunk=1 << 14)
    assert torch.equal(a["labels"], b["labels"])
    assert int((a["codes"].to(torch.int32) - b["codes"].to(torch.int32)).abs().max()) <= 1


def test_labels_follow_schedule():
    cfg = kkgen.LinkConfig(formats=(4, 8, 16, 32, 64), segment_frames=2)
    k = torch.arange(0, 4096 * 20)
    lab = kkgen.symbol_labels(cfg, k)
    M = cfg.format_of_symbols(k)
    assert torch.all(lab.to(torch.int64) < M)
    assert M[0] == 4 and M[4096 * 2] == 8 and M[4096 * 10] == 4
    # roughly uniform
    h = torch.bincount(lab[:4096 * 2].to(torch.int64), minlength=4).double()
    assert float(h.min() / h.max()) > 0.9


def test_white_noise_statistics():
    cfg = kkgen.LinkConfig(esn0_db=10.0, seed=3)
    n = kkgen.gauss_complex(3, torch.arange(1 << 18))
    assert abs(float((n.abs() ** 2).mean()) - 1) < 0.01
    assert abs(float((n * n).mean().abs())) < 0.01                      # circular
    assert abs(cfg.sigma2 - 4 * 0.25 / 10.0) < 1e-15                    # σ² = 4·P_x/(Es/N0) (R14)


def test_codes_bit_identical_for_any_subrange():
    """The generation grid is global (kkgen.GEN_GRID), so a rank's window — any [s0, s1) — has exactly the
    codes of the same samples in a longer stream (the basis of bit-identical multi-GPU shards and of
    single-ingest windows)."""
    lc = kkgen.LinkConfig(formats=(4, 64), segment_frames=1, dl_ps_nm=200000.0, cspr_db=10.0, esn0_db=18.0,
                          seed=5)
    lo, hi = -20000, 3 * kkgen.GEN_GRID + 1000
    full = kkgen.generate(lc, lo, hi)
    for a, b in ((0, 4096), (kkgen.GEN_GRID - 8, kkgen.GEN_GRID + 8), (-20000, -19000), (123456, 600000)):
        sub = kkgen.generate(lc, a, b)
        assert torch.equal(sub["codes"], full["codes"][a - lo:b - lo])
        assert torch.equal(sub["labels"], full["labels"][(a - lo) // 4:(b - lo) // 4])


def test_differential_phase_noise_statistics():
    """P12(v) fixture: φ(t − τ) − φ(t) of a Wiener phase with linewidth Δν has variance 2πΔν·τ (PAPER.md:50
    100 kHz ECL; τ = 0.83 ns), is a function of the global index only (chunk-invariant) and decorrelates
    beyond the delay window."""
    cfg = kkgen.LinkConfig(linewidth_hz=100e3, pn_delay_s=0.83e-9, seed=4)
    n = torch.arange(-(1 << 19), 1 << 19, dtype=torch.int64)
    d = kkgen.differential_phase_noise(cfg, n).numpy()
    var = 2 * math.pi * 100e3 * 0.83e-9
    assert abs(np.var(d) / var - 1) < 0.02 and abs(np.mean(d)) < 0.01 * math.sqrt(var)
    assert np.array_equal(kkgen.differential_phase_noise(cfg, n[1000:2000]).numpy(), d[1000:2000])
    # adjacent samples share two whole increments and the fractional one (weights 1 and √0.32 against 1):
    # correlation (2 + √0.32)/3.32; lag 4 shares none
    c1 = np.corrcoef(d[:-1], d[1:])[0, 1]
    c4 = np.corrcoef(d[:-4], d[4:])[0, 1]
    assert abs(c1 - (2 + math.sqrt(0.32)) / 3.32) < 0.01 and abs(c4) < 0.01
