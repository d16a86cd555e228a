"""kkgen — seeded synthetic KK-link input generator (transmitter + linear channel + ADC).

This module is the ONLY code shared by the oracle side (tests, bench `cpu_baseline`)
and the CUDA side (tests, bench). It holds none of the receiver method's arithmetic:
it builds the *input* of the method — the int16 ADC codes of a minimum-phase KK
photocurrent — and the transmitted labels, exactly as the paper's transmitter and
link describe them (§2 "Experimental setup"):

  * 1 GBaud QAM (4/8/16/32/64) labels from a counter-based hash keyed by
    (seed, global symbol index) — chunk- and shard-invariant;
  * 1 %-roll-off RRC pulse shaping at 4 sps, span 256 symbols;
  * chromatic dispersion as the all-pass exp(+i·β₂L/2·ω²) on the data field,
    ω the optical angular offset from the laser/tone;
  * carrier tone A at the field DC, data at +0.516 GHz;
  * complex AWGN on the field before square law ("white" over the 4 GHz
    simulation band, or "analytic" = positive frequencies only);
  * square-law detection |E|² and an ideal DC-coupled int16 ADC.

Everything is fp64 and device-agnostic torch (CPU for tests; CUDA for the bench's
multi-GiB streams). Random numbers come from a counter-based integer hash so the
sample at global index n never depends on how the stream is chunked or sharded.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch
from scipy.fft import next_fast_len

FS = 4.0e9          # ADC rate ("4 GS/s ADC")
BAUD = 1.0e9        # symbol rate ("1 GBaud")
SPS = 4
F_C = 0.516e9       # tone offset ("carrier tone at 0.516 GHz")
LO_NUM, LO_DEN = 129, 1000   # F_C / FS = 0.129 exactly
ROLLOFF = 0.01      # PAPER.md:50 "1% roll-off"
RRC_SPAN = 256
LAMBDA_M = 1550.51e-9  # PAPER.md:50 ECL wavelength
C_LIGHT = 299792458.0
FRAME_SYMBOLS = 4096  # SURVEY R23 (used only to place the per-segment format schedule)

# ----------------------------------------------------------------------------------
# counter-based hash (murmur3 fmix32 on int64 tensors, overflow-free 32-bit multiply)
# ----------------------------------------------------------------------------------
_M32 = 0xFFFFFFFF


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _M32


def _fmix32(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = _mul32(x, 0x85EBCA6B)
    x = x ^ (x >> 13)
    x = _mul32(x, 0xC2B2AE35)
    x = x ^ (x >> 16)
    return x


def hash_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """32-bit hash of (seed, stream, idx) for int64 idx (any sign)."""
    key = _fmix32(torch.tensor(((seed * 0x9E3779B1) ^ (stream * 0x7F4A7C15)) & _M32,
                               dtype=torch.int64, device=idx.device))
    lo = idx & _M32
    hi = (idx >> 32) & _M32
    h = _fmix32(lo ^ key)
    h = _fmix32(h ^ hi ^ 0x68E31DA4)
    return _fmix32(h ^ key)


def uniform01(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    return (hash_u32(seed, stream, idx).to(torch.float64) + 0.5) * (1.0 / 4294967296.0)


def gauss_complex(seed: int, idx: torch.Tensor) -> torch.Tensor:
    """Unit-variance circular complex Gaussian per index (Box-Muller, E|n|^2 = 1)."""
    u1 = uniform01(seed, 11, idx)
    u2 = uniform01(seed, 12, idx)
    r = torch.sqrt(-torch.log(u1))          # |n|^2 ~ Exp(1)
    ph = 2.0 * math.pi * u2
    return torch.complex(r * torch.cos(ph), r * torch.sin(ph))


# ----------------------------------------------------------------------------------
# transmitter alphabets (labels -> points), SURVEY R13
# ----------------------------------------------------------------------------------
_CROSS32_ROWS = [  # rows Q=+5..-5, columns I=-5..+5; -1 = empty corner
    [-1, 3, 2, 18, 19, -1],
    [6, 14, 10, 26, 30, 22],
    [7, 15, 11, 27, 31, 23],
    [5, 13, 9, 25, 29, 21],
    [4, 12, 8, 24, 28, 20],
    [-1, 0, 1, 17, 16, -1],
]


def tx_alphabet(M: int) -> np.ndarray:
    """points[label] (complex128, unit mean energy) for the transmitter mapper."""
    pts = np.zeros(M, np.complex128)
    gray = lambda i: i ^ (i >> 1)
    if M in (4, 16, 64):
        m = int(round(math.sqrt(M)))
        b2 = int(round(math.log2(m)))
        sc = 1.0 / math.sqrt(2.0 * (M - 1) / 3.0)
        for iI in range(m):
            for iQ in range(m):
                pts[(gray(iI) << b2) | gray(iQ)] = sc * complex(2 * iI - (m - 1), 2 * iQ - (m - 1))
    elif M == 8:
        sc = 1.0 / math.sqrt(6.0)
        for iI in range(4):
            for iQ in range(2):
                pts[(gray(iI) << 1) | iQ] = sc * complex(2 * iI - 3, 2 * iQ - 1)
    elif M == 32:
        sc = 1.0 / math.sqrt(20.0)
        for r, row in enumerate(_CROSS32_ROWS):
            for c, lab in enumerate(row):
                if lab >= 0:
                    pts[lab] = sc * complex(2 * c - 5, 5 - 2 * r)
    else:
        raise ValueError(f"unsupported QAM order {M}")
    return pts


def rrc_taps_tx(rolloff: float = ROLLOFF, span: int = RRC_SPAN, sps: int = SPS) -> np.ndarray:
    """Transmit RRC taps (unit energy, length span*sps+1, centred); textbook RRC impulse response."""
    n = np.arange(-span * sps // 2, span * sps // 2 + 1, dtype=np.float64)
    t = n / sps
    b = rolloff
    h = np.empty_like(t)
    for i, ti in enumerate(t):
        if ti == 0.0:
            h[i] = 1.0 + b * (4.0 / math.pi - 1.0)
        elif abs(abs(4.0 * b * ti) - 1.0) < 1e-12:
            h[i] = (b / math.sqrt(2.0)) * ((1 + 2 / math.pi) * math.sin(math.pi / (4 * b))
                                           + (1 - 2 / math.pi) * math.cos(math.pi / (4 * b)))
        else:
            h[i] = (math.sin(math.pi * ti * (1 - b)) + 4 * b * ti * math.cos(math.pi * ti * (1 + b))) / (
                math.pi * ti * (1 - (4 * b * ti) ** 2))
    return h / math.sqrt(np.sum(h * h))


# ----------------------------------------------------------------------------------
# link configuration
# ----------------------------------------------------------------------------------
@dataclass
class LinkConfig:
    formats: Sequence[int] = (4,)         # QAM order per segment (cycled)
    segment_frames: int = 1 << 30         # frames per segment (format constant within)
    cspr_db: float = 12.0
    esn0_db: Optional[float] = None       # nominal Es/N0 (None = noiseless)
    noise: str = "white"                  # "white" | "analytic"
    dl_ps_nm: float = 0.0                 # accumulated dispersion D*L
    seed: int = 101
    wander_rad: float = 0.0               # optional data-vs-tone phase wander amplitude (CPR fixtures)
    wander_hz: float = 50e3
    # optional physical laser phase noise (CPR fixture P12(v)): the tone and the data share one laser, so after
    # dispersion the data sees φ(t − τ) − φ(t) for a Wiener φ of linewidth Δν ("100 kHz" ECL) and
    # the data-vs-tone delay τ (0.83 ns at 10,000 km)
    linewidth_hz: float = 0.0
    pn_delay_s: float = 0.83e-9
    sideband: int = +1
    adc_bits: int = 15                    # 15 → int16 codes 0..32767 (R20); ≤ 8 → uint8 codes (SPEC S:199's 8-bit ADC)
    label_source: str = "hash"            # "hash" (counter hash per symbol) | "prbs31" (ITU-T O.150 PRBS-31 bit stream)

    @property
    def px(self) -> float:  # mean |x|^2 of the shaped data at 4 sps with unit-energy taps
        return 1.0 / SPS

    @property
    def amp(self) -> float:  # tone amplitude from CSPR = A^2 / P_x
        return math.sqrt(self.px * 10.0 ** (self.cspr_db / 10.0))

    @property
    def sigma2(self) -> float:  # complex noise variance per 4-GS/s sample
        if self.esn0_db is None:
            return 0.0
        return SPS * self.px / 10.0 ** (self.esn0_db / 10.0)

    @property
    def i_clip(self) -> float:  # ADC full scale: fixed by the config (chunk-invariant)
        return (self.amp + 6.0 * math.sqrt(self.px + self.sigma2)) ** 2

    @property
    def adc_max(self) -> int:
        return (1 << self.adc_bits) - 1

    @property
    def adc_scale(self) -> float:
        return self.i_clip / float(self.adc_max)

    @property
    def i_ref(self) -> float:  # expected mean intensity
        return self.amp ** 2 + self.px + self.sigma2

    def format_of_symbols(self, k: torch.Tensor) -> torch.Tensor:
        seg = torch.div(torch.div(k, FRAME_SYMBOLS, rounding_mode="floor"), self.segment_frames,
                        rounding_mode="floor")
        sched = torch.tensor(list(self.formats), dtype=torch.int64, device=k.device)
        return sched[torch.remainder(seg, len(self.formats))]


def esn0_from_osnr(osnr_db: float, cspr_db: float) -> float:
    """E_s/N_0 of the data part at a given OSNR (0.1 nm, single pol) and CSPR."""
    return osnr_db + 10 * math.log10(12.5) - 10 * math.log10(1 + 10 ** (cspr_db / 10))


def beta2_l(dl_ps_nm: float, lam: float = LAMBDA_M) -> float:
    """beta_2 * L in s^2 from accumulated D*L in ps/nm (beta_2 = -D lambda^2 / (2 pi c))."""
    return -(dl_ps_nm * 1e-3) * lam ** 2 / (2 * math.pi * C_LIGHT)


# ----------------------------------------------------------------------------------
# generation
# ----------------------------------------------------------------------------------
def symbol_labels(cfg: LinkConfig, k: torch.Tensor) -> torch.Tensor:
    M = cfg.format_of_symbols(k)
    if cfg.label_source == "prbs31":
        n = k.numel()
        k0 = int(k[0]) if n else 0
        assert n == 0 or bool(torch.equal(k, torch.arange(k0, k0 + n, dtype=torch.int64, device=k.device))), \
            "prbs31 labels: contiguous symbol ranges only"
        return (prbs31_slots(cfg.seed, k0, n, k.device) & (M - 1)).to(torch.uint8)
    assert cfg.label_source == "hash"
    return (hash_u32(cfg.seed, 1, k) & (M - 1)).to(torch.uint8)


# ----------------------------------------------------------------------------------
# PRBS-31 label stream (ITU-T O.150: x^31 + x^28 + 1) — the pattern a real transmitter sends and a real-time
# receiver syncs to (PAPER.md:112 counts BER against the known transmitted sequence). Bit stream b[n]:
# b[n] = b[n−28] ⊕ b[n−31] (n ≥ 31), b[0..30] = the bits of the initial word W0(seed) (LSB = b[0]).
# Symbol k owns the 6-bit slot b[6k .. 6k+5]: slot(k) = Σ_t b[6k+t]·2^t, label(k) = slot(k) & (M(k) − 1).
# Any symbol range is generated independently: the 31-bit window W_n = Σ_i b[n+i]·2^i evolves linearly over GF(2)
# (W_{n+1} = (W_n >> 1) | ((b[n] ⊕ b[n+3]) << 30)), so W_n = A^n·W0 by binary powers of A (jump-ahead).
# ----------------------------------------------------------------------------------
PRBS_MASK31 = (1 << 31) - 1
PRBS_PERIOD = (1 << 31) - 1           # the order of A (x^31 + x^28 + 1 is primitive; 2^31 − 1 is prime)


def prbs31_w0(seed: int) -> int:
    w = ((seed * 0x9E3779B1) & 0xFFFFFFFF) >> 1
    return w if w else 1


def _gf2_apply(cols, w):
    """M·w over GF(2) for the 31×31 matrix with columns cols (ints), w an int or an int64 tensor."""
    if isinstance(w, int):
        r = 0
        for i in range(31):
            if (w >> i) & 1:
                r ^= cols[i]
        return r
    r = torch.zeros_like(w)
    for i in range(31):
        r ^= ((w >> i) & 1) * cols[i]
    return r


def _prbs_step_cols():
    cols = []                                        # A·e_i: shift right by one, new bit 30 = b0 ⊕ b3
    for i in range(31):
        w = 1 << i
        cols.append((w >> 1) | ((((w >> 0) ^ (w >> 3)) & 1) << 30))
    return cols


_PRBS_POW = {}   # n → columns of A^n (powers of two, times the 96-bit block stride)


def prbs31_matrix(n_pow2: int):
    """Columns of A^(2^n_pow2)."""
    if n_pow2 not in _PRBS_POW:
        if n_pow2 == 0:
            _PRBS_POW[0] = _prbs_step_cols()
        else:
            prev = prbs31_matrix(n_pow2 - 1)
            _PRBS_POW[n_pow2] = [_gf2_apply(prev, c) for c in prev]      # (A^m)² column by column
    return _PRBS_POW[n_pow2]


def prbs31_jump(w: int, n: int) -> int:
    """W_n from W_0 = w."""
    j = 0
    while n:
        if n & 1:
            w = _gf2_apply(prbs31_matrix(j), w)
        n >>= 1
        j += 1
    return w


def prbs31_slots(seed: int, k0: int, n: int, device="cpu") -> torch.Tensor:
    """slot(k) for k = k0 … k0 + n − 1 (int64). Blocks of 16 symbols (96 bits) from their 31-bit windows: the first
    block's window by jump-ahead, the others by doubling (W of block b + 2^j = A^(96·2^j)·W of block b)."""
    device = torch.device(device)
    if n == 0:
        return torch.zeros(0, dtype=torch.int64, device=device)
    b0, b1 = k0 // 16, (k0 + n + 15) // 16
    nb = b1 - b0
    # the window at bit 96·b0 (negative positions — the pre-roll before global symbol 0 — by the period 2^31 − 1)
    W = torch.tensor([prbs31_jump(prbs31_w0(seed), (96 * b0) % PRBS_PERIOD)], dtype=torch.int64, device=device)
    j = 0
    while W.numel() < nb:
        # A^(96·2^j) = (A^96)^(2^j): columns from repeated squaring of A^96
        key = ("b96", j)
        if key not in _PRBS_POW:
            if j == 0:
                c96 = [prbs31_jump(1 << i, 96) for i in range(31)]
            else:
                prev = _PRBS_POW[("b96", j - 1)]
                c96 = [_gf2_apply(prev, c) for c in prev]
            _PRBS_POW[key] = c96
        W = torch.cat([W, _gf2_apply(_PRBS_POW[key], W)])
        j += 1
    W = W[:nb]
    m28 = (1 << 28) - 1
    n1 = ((W >> 3) ^ W) & m28                                           # b[31 .. 58]
    W1 = (W >> 28) | (n1 << 3)
    n2 = ((W1 >> 3) ^ W1) & m28                                         # b[59 .. 86]
    W2 = (W1 >> 28) | (n2 << 3)
    n3 = ((W2 >> 3) ^ W2) & m28                                         # b[87 .. 114]
    lo = W | (n1 << 31) | ((n2 & 31) << 59)                             # b[0 .. 63]
    hi = (n2 >> 5) | (n3 << 23)                                         # b[64 .. 114]
    kk = torch.arange(k0, k0 + n, dtype=torch.int64, device=device)
    bi = kk // 16 - b0
    off = 6 * (kk % 16)                                                 # 0 … 90
    lo_k, hi_k = lo[bi], hi[bi]
    # 6 bits starting at off from the 128-bit (hi:lo); lo is a signed int64: mask after the shift
    lo_mask = torch.where(off <= 58, torch.full_like(off, 63), (1 << (64 - off).clamp(min=0, max=6)) - 1)
    from_lo = (lo_k >> off.clamp(max=63)) & lo_mask                     # (arithmetic shift: keep only real bits)
    from_lo = torch.where(off < 64, from_lo, torch.zeros_like(from_lo))
    sh_hi = (64 - off).clamp(min=0)                                     # hi bits land at position 64 − off
    from_hi = torch.where(off >= 64, (hi_k >> (off - 64).clamp(min=0)), (hi_k << sh_hi.clamp(max=63)))
    return (from_lo | from_hi) & 63


def _symbols(cfg: LinkConfig, k: torch.Tensor) -> torch.Tensor:
    lab = symbol_labels(cfg, k).to(torch.int64)
    M = cfg.format_of_symbols(k)
    out = torch.zeros(k.shape, dtype=torch.complex128, device=k.device)
    for m in sorted(set(int(x) for x in cfg.formats)):
        tab = torch.from_numpy(tx_alphabet(m)).to(k.device)
        sel = M == m
        out[sel] = tab[lab[sel]]
    return out


def _data_field(cfg: LinkConfig, s0: int, s1: int, device, guard_sym: int = 1024) -> torch.Tensor:
    """Dispersed, tone-shifted data field x_s[n] for global samples [s0, s1) (multiples of 4)."""
    assert s0 % SPS == 0 and s1 % SPS == 0
    k0, k1 = s0 // SPS - guard_sym, s1 // SPS + guard_sym
    k = torch.arange(k0, k1, dtype=torch.int64, device=device)
    sym = _symbols(cfg, k)
    nfft = next_fast_len((k1 - k0) * SPS)
    u = torch.zeros(nfft, dtype=torch.complex128, device=device)
    u[: (k1 - k0) * SPS: SPS] = sym
    h = rrc_taps_tx()
    half = (len(h) - 1) // 2
    hc = np.zeros(nfft, np.float64)   # circularly centred taps
    hc[: half + 1] = h[half:]
    hc[-half:] = h[:half]
    Hf = torch.fft.fft(torch.from_numpy(hc).to(device))
    nu = torch.fft.fftfreq(nfft, d=1.0 / FS, device=device).to(torch.float64)
    w = 2 * math.pi * (nu + cfg.sideband * F_C)      # optical offset of each data bin
    cd = torch.exp(1j * (beta2_l(cfg.dl_ps_nm) / 2.0) * w * w)
    x = torch.fft.ifft(torch.fft.fft(u) * Hf * cd)
    g = guard_sym * SPS
    x = x[g: g + (s1 - s0)]
    n = torch.arange(s0, s1, dtype=torch.int64, device=device)
    q = torch.remainder(torch.remainder(n, LO_DEN) * LO_NUM, LO_DEN).to(torch.float64)
    ph = cfg.sideband * 2 * math.pi * q / LO_DEN
    if cfg.wander_rad:
        ph = ph + cfg.wander_rad * torch.sin(2 * math.pi * cfg.wander_hz * n.to(torch.float64) / FS)
    if cfg.linewidth_hz:
        ph = ph + differential_phase_noise(cfg, n)
    return x * torch.exp(1j * ph)


def differential_phase_noise(cfg: LinkConfig, n: torch.Tensor) -> torch.Tensor:
    """φ(n − τf_s) − φ(n) for a Wiener laser phase φ with per-sample increments δ_j ~ N(0, 2πΔν/f_s) drawn
    from the counter hash (stream 13): = −(δ_n + … + δ_{n−D+1}) − √r·δ_{n−D}, D = ⌊τf_s⌋, r = τf_s − D.
    Only the increments inside the delay window enter, so the value is local and chunk-invariant; its
    variance is 2πΔν·τ (the Wiener variance over τ)."""
    d = cfg.pn_delay_s * FS
    D = int(math.floor(d))
    r = d - D
    sd = math.sqrt(2 * math.pi * cfg.linewidth_hz / FS)

    def inc(j):
        u1, u2 = uniform01(cfg.seed, 13, j), uniform01(cfg.seed, 14, j)
        return sd * torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)

    out = torch.zeros(n.shape, dtype=torch.float64, device=n.device)
    for m in range(D):
        out -= inc(n - m)
    if r > 0:
        out -= math.sqrt(r) * inc(n - D)
    return out


GEN_GRID = 1 << 18        # samples per generation chunk on the CPU, anchored at global sample 0
GEN_GRID_CUDA = 1 << 24   # on a GPU (fewer launches; invariance holds per device type)


def gen_grid(device) -> int:
    return GEN_GRID_CUDA if torch.device(device).type == "cuda" else GEN_GRID


def generate(cfg: LinkConfig, s0: int, s1: int, device="cpu", chunk: int = GEN_GRID,
             return_field: bool = False):
    """int16 ADC codes for global samples [s0, s1) and labels for symbols [s0/4, s1/4).

    The field is built chunk by chunk on a fixed global grid (chunks [k·G, (k+1)·G), G = gen_grid(device),
    each with the same guard and FFT length), so any sub-range — another chunking, another rank's window —
    yields bit-identical codes on the same device type. (`chunk` is accepted for compatibility and ignored; analytic
    noise, a non-local filter used only for calibration, is generated over [s0, s1) in one piece.)
    Returns dict(codes=int16[s1-s0], labels=uint8[(s1-s0)/4], and the sidecar numbers).
    With return_field=True also the noiseless transmitted field E (complex128).
    """
    device = torch.device(device)
    codes = torch.empty(s1 - s0, dtype=torch.uint8 if cfg.adc_bits <= 8 else torch.int16, device=device)
    fields = []
    analytic = cfg.noise == "analytic" and cfg.sigma2 > 0
    G = gen_grid(device)
    pieces = [(s0, s1)] if analytic else [(c0, c0 + G) for c0 in range((s0 // G) * G, s1, G)]
    for c0, c1 in pieces:
        E = cfg.amp + _data_field(cfg, c0, c1, device)
        a, b = max(c0, s0), min(c1, s1)                # part of the chunk inside [s0, s1)
        E = E[a - c0:b - c0]
        if return_field:
            fields.append(E.clone())
        if cfg.sigma2 > 0:
            if analytic:
                n = torch.arange(c0, c1, dtype=torch.int64, device=device)
                nz = gauss_complex(cfg.seed, n)
                Nf = torch.fft.fft(nz)
                nu = torch.fft.fftfreq(c1 - c0, device=device)
                keep = (nu * cfg.sideband) > 0
                nz = torch.fft.ifft(torch.where(keep, Nf, torch.zeros_like(Nf)))  # same PSD on f>0
            else:
                nz = gauss_complex(cfg.seed, torch.arange(a, b, dtype=torch.int64, device=device))
            E = E + math.sqrt(cfg.sigma2) * nz
        inten = E.real * E.real + E.imag * E.imag
        code = torch.clamp(torch.round(inten * (cfg.adc_max / cfg.i_clip)), 0, cfg.adc_max)
        codes[a - s0: b - s0] = code.to(codes.dtype)
    k = torch.arange(s0 // SPS, s1 // SPS, dtype=torch.int64, device=device)
    out = dict(codes=codes, labels=symbol_labels(cfg, k), adc_scale=cfg.adc_scale,
               adc_offset=0.0, i_ref=cfg.i_ref, amp=cfg.amp, px=cfg.px, sigma2=cfg.sigma2)
    if return_field:
        out["field"] = torch.cat(fields)
    return out


# ----------------------------------------------------------------------------------
# named workloads (BASELINE.json configs)
# ----------------------------------------------------------------------------------
WORKLOADS = {
    "C1": dict(cfg=LinkConfig(formats=(4,), dl_ps_nm=0.0, cspr_db=12.0, seed=101), samples=1 << 16),
    "C2": dict(cfg=LinkConfig(formats=(16,), dl_ps_nm=112000.0, cspr_db=6.0,
                              esn0_db=esn0_from_osnr(17.0, 6.0), seed=201), samples=1 << 22),
    "C3": dict(cfg=LinkConfig(formats=(64,), dl_ps_nm=32000.0, cspr_db=12.0, esn0_db=26.0, seed=301),
               samples=1 << 24),
    "C4": dict(cfg=LinkConfig(formats=(4,), dl_ps_nm=200000.0, cspr_db=12.0, esn0_db=12.0, seed=401),
               samples=1 << 26),
    "C5": dict(cfg=LinkConfig(formats=(4, 8, 16, 32, 64), segment_frames=256, dl_ps_nm=32000.0,
                              cspr_db=12.0, esn0_db=26.0, seed=501, label_source="prbs31"), samples=1 << 32),
}
