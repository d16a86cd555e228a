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


def test_prbs31_labels_follow_the_recurrence():
    """ITU-T O.150 PRBS-31 (x^31 + x^28 + 1): kkgen's block/jump-ahead generation equals the plain bit-by-bit
    recurrence b[n] = b[n−28] ⊕ b[n−31] from the seed's initial word, for arbitrary symbol ranges (slot(k) = bits
    6k … 6k+5, LSB first)."""
    for seed in (7, 501):
        w = kkgen.prbs31_w0(seed)
        b = [(w >> i) & 1 for i in range(31)]
        while len(b) < 6 * 5000 + 64:
            b.append(b[-28] ^ b[-31])
        ref = torch.tensor([sum(b[6 * k + t] << t for t in range(6)) for k in range(5000)])
        for k0, n in ((0, 5000), (7, 333), (16 * 40 + 5, 1200), (4999, 1)):
            assert torch.equal(kkgen.prbs31_slots(seed, k0, n), ref[k0:k0 + n])


def test_prbs31_period_and_negative_positions():
    """A has order 2^31 − 1 (a primitive polynomial; 2^31 − 1 is prime, so no proper divisor returns to W0);
    negative symbol indices (the generator's pre-roll) continue the same periodic stream."""
    w = kkgen.prbs31_w0(3)
    assert kkgen.prbs31_jump(w, kkgen.PRBS_PERIOD) == w
    assert kkgen.prbs31_jump(w, 1) != w and kkgen.prbs31_jump(w, kkgen.PRBS_PERIOD - 1) != w
    a = kkgen.prbs31_slots(3, -100, 300)
    assert torch.equal(a[100:], kkgen.prbs31_slots(3, 0, 200))
    # slot(−1) = bits −6 … −1 = bits P−6 … P−1 of one period
    tail = kkgen.prbs31_jump(w, kkgen.PRBS_PERIOD - 6)
    assert int(a[99]) == (tail & 63)


def test_prbs31_link_labels_are_balanced_and_generated():
    cfg = kkgen.LinkConfig(formats=(16, 64), segment_frames=1, seed=11, label_source="prbs31")
    k = torch.arange(0, 4 * 4096, dtype=torch.int64)
    lab = kkgen.symbol_labels(cfg, k).numpy()
    assert lab[:4096].max() <= 15 and lab[4096:8192].max() <= 63
    assert abs(np.mean(np.unpackbits(lab[4096:8192, None], axis=1)[:, 2:]) - 0.5) < 0.02
    g = kkgen.generate(cfg, -16640, 16384 + 16640)
    assert torch.equal(g["labels"], kkgen.symbol_labels(cfg, torch.arange(-4160, 8256, dtype=torch.int64)))
