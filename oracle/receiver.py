"""The KK receive chain, step by step in fp64 (oracle; TEST INFRASTRUCTURE ONLY).

Steps O1–O11 follow PAPER.md:82 (§2, DSP chain of Fig. 1b) in the paper's order, with
the north-star changes (BASELINE.json: carrier removal, block-adaptive FIR absorbing CD,
carrier-phase recovery) and the readings R1–R27 of SURVEY.md §8(c):

  O1  I[n] = s·(c[n] − o)                                   PAPER.md:82 "converts the samples to floating point"
  O2  a[n] = ½·ln max(I[n], ε), ε = clamp_rel·I_ref         PAPER.md:82 "square-root and logarithm"; R7
  O3  φ = σ·Hilbert(a) by 1024-pt OLS, hop 512, centre kept   PAPER.md:82 "pair of 1024-point 100% overlap-save FFTs"; R1, R2
  O4  E[n] = √max(I,ε)·e^{iφ[n]}                              PAPER.md:82 "combined with the amplitude ... reconstruct the optical field"
  O5  A_f = mean_{n∈f} E[n];  e[n] = E[n] − A_{f(n)}           BASELINE.json north_star "carrier removal"; R8
  O6  b[n] = e[n]·exp(−2πiσ·((lo_num·n) mod lo_den)/lo_den)    PAPER.md:82 "downshifted to DC"; R9
  O7  y[m] = Σ_{j=−512}^{512} h[j]·b[2m − j]                    PAPER.md:82 "static equalization and downsampling from 4 to 2"; R4, R5, R6
  O8  per-frame widely-linear DD least-squares FIR              PAPER.md:82 "adaptive ... DDLMS widely-linear"; north_star; R10, R25, R27
  O9  CPR: ϑ_b = arg Σ_{k∈b} v_k·conj(D(v_k)); z = v·e^{−iϑ_b}   north_star "carrier-phase recovery"; R12
  O10 decisions and error counts                             PAPER.md:82 "decisions ... are demapped"; PAPER.md:112
  O11 Q = 20·log10(√2·erfcinv(2·BER))                        PAPER.md:112; SPEC S:71 (theory.q_from_ber)

  O3u (upsample = 2, SPEC S:277/S:375 upsample_factor — "KK in-principle benefits
      from digital upsampling before the nonlinear sqrt/log"; DESIGN.md §3 "KK upsampling"): per Hilbert
      block j, I is interpolated to 8 sps by the half-band filter f over the block's 2048-sample window,
      O2–O4 run at 8 sps (2048-pt Hilbert, same time span as the 1024-pt one at 4 sps), and E at 4 sps is
      the half-band decimation of the block's own 8-sps field.

Library primitives used as single steps: numpy.fft (O3), scipy.signal.fftconvolve (O7),
numpy.linalg.lstsq (CD-init fit), dense Φ̃ᴴΦ̃ and numpy.linalg.cholesky/solve (O8),
brute-force nearest point (O8–O10).
"""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
from scipy import signal

from .constellation import constellation, nearest, popcount

C_LIGHT = 299792458.0


@dataclass
class OracleConfig:
    fs_hz: float = 4e9
    baud_hz: float = 1e9
    lo_num: int = 129                 # f_c / f_s = 129/1000 ("0.516 GHz" at 4 GS/s)
    lo_den: int = 1000
    sideband: int = +1                # data above the tone (R2, R3)
    rolloff: float = 0.01             # PAPER.md:50 "1% roll-off"
    rrc_span_sym: int = 256           # R4
    hilbert_n: int = 1024             # PAPER.md:82 "1024-point"
    hilbert_hop: int = 512            # R1
    frame_symbols: int = 4096         # R23
    eq_taps: int = 0                  # 0 = tap-count rule
    eq_widely_linear: bool = True     # PAPER.md:82 "widely-linear"
    eq_ridge: float = 1e-3            # R10
    cpr_window: int = 256             # R12
    dispersion_ps_per_nm: float = 0.0
    lambda_m: float = 1550.51e-9
    adc_scale: float = 1.0
    adc_offset: float = 0.0
    ref_intensity: float = 1.0
    clamp_rel: float = 1e-12          # R7
    p0_min_rel: float = 1e-20         # silent-frame rule: AGC power ≤ p0_min_rel·I_ref ⇒ bad frame, z = 0
    formats: Sequence[int] = (4,)     # per-segment QAM order (R26)
    segment_frames: int = 1 << 30
    # paper arrangement: eq_mode "ddlms" folds the CD inverse
    # into the static filter and equalizes with the 4-tap T/2-spaced widely-linear DDLMS
    static_cd: bool = False           # block_ls after the paper's static RRC × CD-inverse filter (NEXT-2): θ₀ = spike
    eq_mode: str = "block_ls"         # "block_ls" (north star, default) | "ddlms" (paper, restart grid) |
                                      # "ddlms_seq" (paper, one recursion in stream order: the definition)
    ddlms_mu_warm: float = 2e-3       # step size over the first half of the warm-up
    ddlms_mu_mid: float = 5e-4        # … over the second half of the warm-up
    ddlms_mu: float = 2.5e-4          # step size over the kept symbols (SPEC S:377 schedule end)
    ddlms_block: int = 512            # symbols kept per DDLMS restart (global grid)
    ddlms_warmup: int = 1024          # symbols run before each block from the centre-spike state
    ddlms_seq_mu0: float = 1e-3       # sequential form: μ over the first ddlms_seq_switch symbols
    ddlms_seq_switch: int = 10000     # … then ddlms_mu (2.5e-4)
    # KK upsampling (O3u): 1 = the paper's 4-sps chain; 2 = interpolate I to 8 sps before sqrt/log
    upsample: int = 1
    halfband_t: int = 8               # odd half-band taps per side (f[±1], f[±3], …, f[±(2T−1)])
    halfband_beta: float = 10.0       # Kaiser window β

    @property
    def sps(self) -> int:
        return int(round(self.fs_hz / self.baud_hz))

    @property
    def frame_samples(self) -> int:
        return self.frame_symbols * self.sps

    def fmt_of_frame(self, f: int) -> int:
        return int(self.formats[(f // self.segment_frames) % len(self.formats)])


# ------------------------------------------------------------------------------------------
# init-time constants
# ------------------------------------------------------------------------------------------
def rrc_taps(cfg: OracleConfig) -> np.ndarray:
    """Unit-energy RRC, span `rrc_span_sym` symbols at 4 sps, index j = −span·2 .. +span·2 (R4)."""
    sps = cfg.sps
    half = cfg.rrc_span_sym * sps // 2
    b = cfg.rolloff
    h = np.zeros(2 * half + 1)
    for idx in range(2 * half + 1):
        t = (idx - half) / sps                     # in symbol periods
        if t == 0:
            h[idx] = 1 - b + 4 * b / math.pi
        elif abs(4 * b * abs(t) - 1) < 1e-12:
            h[idx] = b / math.sqrt(2) * ((1 + 2 / math.pi) * math.sin(math.pi / (4 * b))
                                         + (1 - 2 / math.pi) * math.cos(math.pi / (4 * b)))
        else:
            num = math.sin(math.pi * t * (1 - b)) + 4 * b * t * math.cos(math.pi * t * (1 + b))
            h[idx] = num / (math.pi * t * (1 - (4 * b * t) ** 2))
    return h / np.sqrt(np.sum(h ** 2))


def beta2L(cfg: OracleConfig) -> float:
    """β₂·L (s²) from accumulated dispersion D·L (ps/nm): β₂ = −D·λ²/(2πc)."""
    dl_si = cfg.dispersion_ps_per_nm * 1e-12 / 1e-9
    return -dl_si * cfg.lambda_m ** 2 / (2 * math.pi * C_LIGHT)


def tap_count(cfg: OracleConfig) -> int:
    """L = 2·⌈τ_max/(T/2)⌉ + 7, τ_max = |β₂L|·2π·(f_c + (1+β)R_s/2) (SURVEY §8(a) tap-count rule); with the static
    CD inverse in the MF (static_cd) the FIR only trims the residual: L = 5 unless set."""
    if cfg.eq_taps:
        return cfg.eq_taps
    if cfg.static_cd and cfg.eq_mode == "block_ls":
        return 5
    f_c = cfg.fs_hz * cfg.lo_num / cfg.lo_den
    tau = abs(beta2L(cfg)) * 2 * math.pi * (f_c + (1 + cfg.rolloff) * cfg.baud_hz / 2)
    return 2 * int(math.ceil(tau / (0.5 / cfg.baud_hz) - 1e-12)) + 7


def cd_init_taps(cfg: OracleConfig) -> np.ndarray:
    """w_cd = argmin Σ_ν |Σ_j w_j e^{−i2πνj/(2R_s)} − C(ν)|², j = −K..K, 2001 ν on ±(1+β)R_s/2,
    C(ν) = exp(−i·(β₂L/2)·(2π(ν + σf_c))²) — the CD inverse referenced to the tone."""
    L = tap_count(cfg)
    K = (L - 1) // 2
    f_c = cfg.fs_hz * cfg.lo_num / cfg.lo_den
    nu = np.linspace(-(1 + cfg.rolloff) * cfg.baud_hz / 2, (1 + cfg.rolloff) * cfg.baud_hz / 2, 2001)
    j = np.arange(-K, K + 1)
    A = np.exp(-2j * np.pi * np.outer(nu, j) / (2 * cfg.baud_hz))
    C = np.exp(-1j * (beta2L(cfg) / 2) * (2 * np.pi * (nu + cfg.sideband * f_c)) ** 2)
    w, *_ = np.linalg.lstsq(A, C, rcond=None)
    return w


# ------------------------------------------------------------------------------------------
# O1–O7: sample-rate stages on a contiguous global range
# ------------------------------------------------------------------------------------------
def o1_intensity(codes: np.ndarray, cfg: OracleConfig) -> np.ndarray:
    return cfg.adc_scale * (codes.astype(np.float64) - cfg.adc_offset)


def o2_front_end(I: np.ndarray, cfg: OracleConfig):
    eps = cfg.clamp_rel * cfg.ref_intensity
    clamped = I < eps
    Ic = np.maximum(I, eps)
    return 0.5 * np.log(Ic), np.sqrt(Ic), clamped


def o3_hilbert_ols(a: np.ndarray, g0: int, out0: int, out1: int, cfg: OracleConfig) -> np.ndarray:
    """φ[n] for global n ∈ [out0, out1) from a over global [g0, g0+len(a)). Block j keeps
    [hop·j, hop·j+hop) of the circular Hilbert of a[hop·j − (N−hop)/2, +N); multiplier −i·sgn(q),
    zero at q ∈ {0, N/2} (R1, R2)."""
    N, hop = cfg.hilbert_n, cfg.hilbert_hop
    lead = (N - hop) // 2
    assert out0 % hop == 0 and out1 % hop == 0
    q = np.arange(N)
    mult = np.where((q > 0) & (q < N // 2), -1j, np.where(q > N // 2, 1j, 0.0))
    phi = np.empty(out1 - out0)
    for jb in range(out0 // hop, out1 // hop):
        s = hop * jb - lead - g0
        assert s >= 0 and s + N <= len(a), "Hilbert input outside the provided range"
        blk = np.fft.ifft(np.fft.fft(a[s:s + N]) * mult).real
        phi[hop * jb - out0: hop * jb - out0 + hop] = blk[lead:lead + hop]
    return cfg.sideband * phi


def halfband_taps(cfg: OracleConfig):
    """Half-band filter f[k], k = −(2T−1)…2T−1 at 8 sps (DESIGN.md §3 "KK upsampling"): f[0] = ½,
    f[even ≠ 0] = 0, f[odd k] = ½·sinc(k/2)·kaiser_β(k), the odd taps rescaled to sum to ½ (unit DC gain).
    Interpolation uses 2f on the odd phase, decimation uses f."""
    T = cfg.halfband_t
    k = np.arange(-(2 * T - 1), 2 * T)
    f = 0.5 * np.sinc(k / 2.0) * np.kaiser(len(k), cfg.halfband_beta)
    odd = (k % 2) != 0
    f[~odd] = 0.0
    f[odd] *= 0.5 / f[odd].sum()
    f[k == 0] = 0.5
    return k, f


def o3u_field_upsampled(I: np.ndarray, g0: int, out0: int, out1: int, cfg: OracleConfig) -> np.ndarray:
    """E[n] for global 4-sps n ∈ [out0, out1) with 2× KK upsampling, I over global [g0, g0 + len(I)).

    For 4-sps Hilbert block j (outputs [512j, 512j + 512)) the 8-sps window is P ∈ [1024j − 512, 1024j + 1536):
      I₂[P] = I[P/2] (P even);  I₂[P] = Σ_{k odd} 2f[k]·I[(P − k)/2] (P odd)          interpolation
      a₂ = ½·ln max(I₂, ε);  φ₂ = σ·IFFT₂₀₄₈(FFT₂₀₄₈(a₂)·(−i·sgn q))  (q = 0, 1024 → 0)    O2, O3 at 8 sps
      E₂ = √max(I₂, ε)·e^{iφ₂}                                                       O4 at 8 sps
      E[n] = Σ_k f[k]·E₂[2n − k]   (E₂ of the block's own window)                     decimation
    """
    assert cfg.upsample == 2
    N, hop = 2 * cfg.hilbert_n, 2 * cfg.hilbert_hop
    lead = (N - hop) // 2
    h4 = cfg.hilbert_hop
    assert out0 % h4 == 0 and out1 % h4 == 0
    eps = cfg.clamp_rel * cfg.ref_intensity
    k, f = halfband_taps(cfg)
    q = np.arange(N)
    mult = np.where((q > 0) & (q < N // 2), -1j, np.where(q > N // 2, 1j, 0.0))
    E = np.empty(out1 - out0, complex)
    odd_taps = [(int(kt), float(ft)) for kt, ft in zip(k, f) if kt % 2 != 0]
    for jb in range(out0 // h4, out1 // h4):
        P = np.arange(hop * jb - lead, hop * jb - lead + N)          # 8-sps window positions
        I2 = np.empty(N)
        ev = (P % 2) == 0
        I2[ev] = I[P[ev] // 2 - g0]
        Po = P[~ev]
        I2[~ev] = sum(2.0 * ft * I[(Po - kt) // 2 - g0] for kt, ft in odd_taps)
        Ic = np.maximum(I2, eps)
        a2 = 0.5 * np.log(Ic)
        phi2 = cfg.sideband * np.fft.ifft(np.fft.fft(a2) * mult).real
        E2 = np.sqrt(Ic) * np.exp(1j * phi2)
        n = np.arange(h4 * jb, h4 * jb + h4)
        E[n - out0] = 0.5 * E2[2 * n - P[0]] + sum(ft * E2[2 * n - kt - P[0]] for kt, ft in odd_taps)
    return E


def o5_carrier_removal(E: np.ndarray, e0: int, cfg: OracleConfig):
    """A_f = mean of E over frame f (global 16384-sample grid); e = E − A_{f(n)} (R8)."""
    F = cfg.frame_samples
    assert e0 % F == 0 and len(E) % F == 0
    A = E.reshape(-1, F).mean(axis=1)
    return E - np.repeat(A, F), A


def o6_mixer(e: np.ndarray, e0: int, cfg: OracleConfig) -> np.ndarray:
    n = np.arange(e0, e0 + len(e), dtype=np.int64)
    q = np.mod(cfg.lo_num * np.mod(n, cfg.lo_den), cfg.lo_den)
    return e * np.exp(-2j * np.pi * cfg.sideband * q / cfg.lo_den)


def o7_matched_filter(b: np.ndarray, b0: int, m0: int, m1: int, h: np.ndarray) -> np.ndarray:
    """y[m] = Σ_j h[j]·b[2m − j] for m ∈ [m0, m1) (exact decimated linear convolution; R6)."""
    half = (len(h) - 1) // 2
    c = signal.fftconvolve(b, h, mode="full")          # c[i] = Σ_t h_arr[t]·b[i − t]
    n = 2 * np.arange(m0, m1, dtype=np.int64)
    assert n[0] - half >= b0 and n[-1] + half < b0 + len(b), "MF input outside provided range"
    return c[n - b0 + half]


def static_filter_taps(cfg: OracleConfig) -> np.ndarray:
    """Paper arrangement ("frequency-domain static equalization ... multiplication with an
    offline-optimized filter"): RRC matched filter × CD inverse referenced to the carrier,
    defined on the 4096-point grid and truncated to the 1025 taps j = −512..512:
        h_cd[j] = (1/4096)·Σ_k H_rrc[k]·C(ν_k)·e^{2πi·kj/4096},  C(ν) = exp(−i(β₂L/2)(2π(ν + σf_c))²),
    ν_k the baseband frequency of FFT bin k at 4 GS/s."""
    h = rrc_taps(cfg)
    N = 4096
    half = (len(h) - 1) // 2
    hc = np.zeros(N)
    hc[:half + 1] = h[half:]
    hc[-half:] = h[:half]
    nu = np.fft.fftfreq(N, d=1.0 / cfg.fs_hz)
    f_c = cfg.fs_hz * cfg.lo_num / cfg.lo_den
    C = np.exp(-1j * (beta2L(cfg) / 2) * (2 * np.pi * (nu + cfg.sideband * f_c)) ** 2)
    full = np.fft.ifft(np.fft.fft(hc) * C)
    j = np.arange(-half, half + 1)
    return full[j % N]


def o8_ddlms_block(y: np.ndarray, m0: int, n0: int, nwarm: int, nkeep: int, M, cfg: OracleConfig,
                   decide=nearest):
    """4-tap T/2-spaced widely-linear DDLMS, restarted per block.
    Symbols n = n0 .. n0 + nwarm + nkeep − 1 (global); x_n = [u[2n+1], u[2n], u[2n−1], u[2n−2]] with
    u = g·y, g = (mean_n |y[2n]|²)^(−½) (AGC over the block and its warm-up);
    out_n = wᵀx_n + vᵀconj(x_n), d_n = D(out_n), e_n = d_n − out_n, w += μ·e·conj(x), v += μ·e·x;
    w starts as the centre spike on u[2n], v = 0 (and stays 0 when eq_widely_linear is False);
    μ = ddlms_mu_warm over the first half of the warm-up, ddlms_mu_mid over its second half, ddlms_mu after.
    M is the QAM order of every symbol (an int, or one per symbol: each symbol is decided in its own frame's
    format, "d[n] = nearest constellation point"). Returns the outputs of the nkeep kept symbols
    (before each one's update). `decide` is the hard
    decision D (default: brute-force nearest point; tests substitute a recording/flipping wrapper)."""
    nn = np.arange(n0, n0 + nwarm + nkeep)
    centres = y[2 * nn - m0]
    P = np.mean(np.abs(centres) ** 2)
    g = 1.0 / math.sqrt(P) if P > 0 else 1.0
    w = np.array([0, 1, 0, 0], complex)
    v = np.zeros(4, complex)
    out = np.zeros(nkeep, complex)
    Ms = np.broadcast_to(np.asarray(M), (len(nn),))
    for i, n in enumerate(nn):
        x = g * y[2 * n - m0 + np.array([1, 0, -1, -2])]
        o = np.dot(w, x) + np.dot(v, np.conj(x))
        d, _ = decide(np.array([o]), int(Ms[i]))
        e = d[0] - o
        mu = cfg.ddlms_mu_warm if i < nwarm // 2 else cfg.ddlms_mu_mid if i < nwarm else cfg.ddlms_mu
        if i >= nwarm:
            out[i - nwarm] = o
        w = w + mu * e * np.conj(x)
        if cfg.eq_widely_linear:
            v = v + mu * e * x
    return out


def o8_ddlms_sequential(y: np.ndarray, m0: int, n0: int, Ms: np.ndarray, cfg: OracleConfig, state=None):
    """The paper's 4-tap T/2-spaced widely-linear DDLMS as ONE recursion in stream order ("four-tap
    adaptive time-domain DDLMS widely-linear equalizer", "sequential time-domain algorithms such as DDLMS";
    SPEC S:351 "Sequential over n; state' carries taps for the next frame in stream order"; S:377 w = centre
    spike, v = 0, μ = 1e-3 then 2.5e-4 after 10^4 symbols). Symbols n = n0 … n0 + len(Ms) − 1 (global), QAM
    order Ms[i] per symbol:
        x_n = g·[y[2n+1], y[2n], y[2n−1], y[2n−2]],  out_n = wᵀx_n + vᵀconj(x_n),  d_n = D(out_n),
        e_n = d_n − out_n,  w += μ_n·e_n·conj(x_n),  v += μ_n·e_n·x_n   (v ≡ 0 when eq_widely_linear is False)
    with μ_n = ddlms_seq_mu0 for the stream's first ddlms_seq_switch symbols, ddlms_mu after. `state` = None
    starts the stream: w = [0, 1, 0, 0] (the spike on the symbol centre y[2n], the restart form's convention),
    v = 0, and the gain g = (mean |y[2n]|² over the stream's first frame)^(−½), kept for the stream (the
    paper states no AGC; a fixed input normalisation is the reading). Returns (outputs before each update,
    state') with state' = dict(w, v, g, count) for the next call."""
    nsym = len(Ms)
    if state is None:
        c = y[2 * np.arange(n0, n0 + min(nsym, cfg.frame_symbols)) - m0]
        P = float(np.mean(np.abs(c) ** 2))
        state = dict(w=np.array([0, 1, 0, 0], complex), v=np.zeros(4, complex),
                     g=1.0 / math.sqrt(P) if P > 0 else 1.0, count=0)
    w, v, g, cnt = state["w"].copy(), state["v"].copy(), state["g"], state["count"]
    tabs = {}
    out = np.zeros(nsym, complex)
    taps = np.array([1, 0, -1, -2])
    for i in range(nsym):
        M = int(Ms[i])
        if M not in tabs:
            tabs[M] = constellation(M)[0]
        pts = tabs[M]
        x = g * y[2 * (n0 + i) - m0 + taps]
        o = np.dot(w, x) + np.dot(v, np.conj(x))
        d = pts[np.argmin(np.abs(pts - o))]                 # D: brute-force nearest point
        e = d - o
        mu = cfg.ddlms_seq_mu0 if cnt < cfg.ddlms_seq_switch else cfg.ddlms_mu
        out[i] = o
        w = w + mu * e * np.conj(x)
        if cfg.eq_widely_linear:
            v = v + mu * e * x
        cnt += 1
    return out, dict(w=w, v=v, g=g, count=cnt)


def _symbol_formats(n0: int, count: int, cfg: OracleConfig) -> np.ndarray:
    """QAM order of global symbols n0 … n0 + count − 1 (format per frame, R26)."""
    fr = np.arange(n0, n0 + count) // cfg.frame_symbols
    return np.array([cfg.fmt_of_frame(int(f)) for f in fr])


# ------------------------------------------------------------------------------------------
# O8–O10: per-frame equalizer, CPR, decisions
# ------------------------------------------------------------------------------------------
def o8_equalize_frame(yf: np.ndarray, K: int, w_cd: np.ndarray, M: int, cfg: OracleConfig,
                      widely_linear: Optional[bool] = None, decide=nearest):
    """One frame. yf = y[2k0 − K, 2k0 + 2F − 2 + K] (length 2F − 1 + 2K). Returns (u, info) with
    u the unbiased pass-2 output of the frame's F symbols (SURVEY §8(a) a7 steps 1–7). `decide` is the
    hard decision D used for the training (pass-1) and unbias decisions (default: brute-force nearest
    point; tests substitute a recording/flipping wrapper)."""
    wl = cfg.eq_widely_linear if widely_linear is None else widely_linear
    L = 2 * K + 1
    F = (len(yf) - 2 * K + 1) // 2
    # (1) regressor φ̃_k = [y[2k − j]]_{j=−K..K} ‖ conj(·)
    kk = np.arange(F)
    idx = 2 * kk[:, None] - np.arange(-K, K + 1)[None, :] + K
    U = yf[idx]
    Phi = np.concatenate([U, np.conj(U)], axis=1) if wl else U
    n_par = Phi.shape[1]
    # (2) θ₀ = [w_cd; 0]
    th0 = np.concatenate([w_cd, np.zeros(L, complex)]) if wl else w_cd.astype(complex)
    # (3) AGC: g = (mean |φ̃ᵀθ₀|²)^(−½) ; θ₀ ← g·θ₀   (R25)
    y0 = Phi @ th0
    P0 = np.mean(np.abs(y0) ** 2)
    if not (P0 > cfg.p0_min_rel * cfg.ref_intensity and np.isfinite(P0)):
        # no signal power to train on (e.g. the tone without modulation): a bad frame, z = 0, decisions D(0)
        return np.zeros(F, complex), dict(theta0=th0, theta1=th0, g=1.0, gamma=0.0, bad=True, silent=True,
                                          R=None, p=None, lam=0.0)
    bad = False
    g = 1.0 / math.sqrt(P0)
    th0 = g * th0
    # (4) pass 1 and decisions
    y0 = Phi @ th0
    d, _ = decide(y0, M)
    # (5) DD least squares with ridge toward θ₀: θ₁ = (R + λI)^(−1)(p + λθ₀), λ = ridge·tr(R)/(2L)
    R = Phi.conj().T @ Phi
    p = Phi.conj().T @ d
    lam = cfg.eq_ridge * np.real(np.trace(R)) / n_par
    Areg = R + lam * np.eye(n_par)
    try:
        Lc = np.linalg.cholesky(Areg)
        th1 = np.linalg.solve(Lc.conj().T, np.linalg.solve(Lc, p + lam * th0))
        if not np.all(np.isfinite(th1)):
            raise np.linalg.LinAlgError
    except np.linalg.LinAlgError:
        th1, bad = th0, True
    # (6) pass 2
    y1 = Phi @ th1
    # (7) gain unbias (R27)
    u, gam, ok = o8_unbias(y1, M, decide)
    bad = bad or not ok
    return u, dict(theta0=th0, theta1=th1, g=g, gamma=gam, bad=bad, R=R, p=p, lam=lam)


def o8_unbias(y1: np.ndarray, M: int, decide=nearest):
    """Gain unbias (R27): γ = Σ y¹·conj(D(y¹)) / Σ|D(y¹)|², u = y¹/|γ|.
    The LS (MMSE) solution shrinks the constellation by the factor |γ| < 1 under noise; dividing by |γ|
    restores unit decision-directed gain (the phase of γ is left to the CPR). Returns (u, γ, ok); ok is
    False (and u = y¹) when |γ| is zero or not finite (counted as a bad frame by the caller)."""
    d1, _ = decide(y1, M)
    gam = np.sum(y1 * np.conj(d1)) / np.sum(np.abs(d1) ** 2)
    if abs(gam) > 0 and np.isfinite(abs(gam)):
        return y1 / abs(gam), gam, True
    return y1, gam, False


def o9_cpr(u: np.ndarray, M: int, W: int, decide=nearest):
    """ϑ_b = arg Σ_{k∈b} u_k·conj(D(u_k)) per W-symbol window aligned to the frame; z = u·e^{−iϑ_b} (R12)."""
    d, _ = decide(u, M)
    s = (u * np.conj(d)).reshape(-1, W).sum(axis=1)
    th = np.where(s != 0, np.angle(s), 0.0)
    return u * np.repeat(np.exp(-1j * th), W), th


# ------------------------------------------------------------------------------------------
# the whole chain over a shard
# ------------------------------------------------------------------------------------------
def halo(cfg: OracleConfig) -> int:
    """Samples needed on each side of the core: one neighbour frame + half a Hilbert block (+ 16 for the
    half-band interpolator's reach when upsample = 2: T ≤ 16 4-sps samples, kept a multiple of 16)."""
    h = cfg.frame_samples + (cfg.hilbert_n - cfg.hilbert_hop) // 2
    if cfg.upsample == 2:
        assert cfg.halfband_t <= 16
        h += 16
    return h


def receive(codes: np.ndarray, first: int, n: int, cfg: OracleConfig, ref: Optional[np.ndarray] = None,
            keep: bool = True) -> dict:
    """Run O1–O10 on the core [first, first+n) given codes for [first − H, first + n + H)."""
    F = cfg.frame_samples
    H = halo(cfg)
    assert first % F == 0 and n % F == 0 and n > 0
    assert len(codes) == n + 2 * H
    g0 = first - H
    # O1, O2
    I = o1_intensity(np.asarray(codes), cfg)
    a, amp, clamped = o2_front_end(I, cfg)
    # O3, O4 over core ± one frame
    e0, e1 = first - F, first + n + F
    if cfg.upsample == 2:
        phi = None
        E = o3u_field_upsampled(I, g0, e0, e1, cfg)
    else:
        assert cfg.upsample == 1
        phi = o3_hilbert_ols(a, g0, e0, e1, cfg)
        E = amp[e0 - g0:e1 - g0] * np.exp(1j * phi)
    # O5, O6
    e, A = o5_carrier_removal(E, e0, cfg)
    b = o6_mixer(e, e0, cfg)
    # O7 over the 2-sps range the frames need
    ddlms = cfg.eq_mode == "ddlms"
    seq = cfg.eq_mode == "ddlms_seq"
    assert cfg.eq_mode in ("block_ls", "ddlms", "ddlms_seq")
    L = tap_count(cfg)
    K = (L - 1) // 2
    if ddlms:
        K = 2 * cfg.ddlms_warmup + 2                   # warm-up reaches 2W + 2 samples before the core
    if seq:
        K = 2                                          # taps y[2n+1] … y[2n−2]
    m0, m1 = first // 2 - K, (first + n) // 2 + K
    h = static_filter_taps(cfg) if (ddlms or seq or cfg.static_cd) else rrc_taps(cfg)
    y = o7_matched_filter(b, e0, m0, m1, h)
    # O8–O10 per frame
    # θ₀: the CD-inverse fit referenced to the carrier; the centre spike when the static filter already inverts CD
    w_cd = cd_init_taps(dataclasses.replace(cfg, dispersion_ps_per_nm=0.0) if cfg.static_cd else cfg)
    Fs = cfg.frame_symbols
    nfr = n // F
    z = np.zeros(n // cfg.sps, complex)
    dec = np.zeros(n // cfg.sps, np.int64)
    counts = dict(sym=np.zeros(5, np.int64), sym_err=np.zeros(5, np.int64), bits=np.zeros(5, np.int64),
                  bit_err=np.zeros(5, np.int64), clamped=int(clamped[H:H + n].sum()), frames=nfr,
                  dead_frames=0, bad_frames=0)
    frame_err = np.zeros((nfr, 2), np.int64)           # per-frame (symbol, bit) errors (PAPER.md:112 bins)
    infos = []
    seq_state = None                                   # ddlms_seq: equalizer state carried in stream order
    for fi in range(nfr):
        f = first // F + fi
        M = cfg.fmt_of_frame(f)
        k0 = fi * Fs                                    # local symbol index
        dead = bool(np.all(clamped[H + fi * F: H + (fi + 1) * F]))
        if dead:
            counts["dead_frames"] += 1
            zf = np.zeros(Fs, complex)
            _, lab = nearest(np.full(Fs, -1e-9 - 1e-9j), M)   # D(0) with ties to the lower level (R15)
            info = dict(dead=True, bad=False)
        elif seq:
            kg0 = first // cfg.sps + k0
            zf, seq_next = o8_ddlms_sequential(y, m0, kg0, np.full(Fs, M), cfg, seq_state)
            seq_state = seq_next
            info = dict(dead=False, bad=False)
            _, lab = nearest(zf, M)
        elif ddlms:
            B, W = cfg.ddlms_block, cfg.ddlms_warmup
            kg0 = first // cfg.sps + k0                 # global symbol index of the frame start
            zf = np.concatenate([o8_ddlms_block(y, m0, kg0 + bb - W, W, B, _symbol_formats(kg0 + bb - W, W + B, cfg),
                                                cfg) for bb in range(0, Fs, B)])
            info = dict(dead=False, bad=False)
            _, lab = nearest(zf, M)
        else:
            yf = y[2 * k0: 2 * k0 + 2 * Fs - 1 + 2 * K]
            u, info = o8_equalize_frame(yf, K, w_cd, M, cfg)
            counts["bad_frames"] += int(info["bad"])
            if info.get("silent"):
                zf = np.zeros(Fs, complex)
                _, lab = nearest(np.full(Fs, -1e-9 - 1e-9j), M)   # D(0) with ties to the lower level (R15)
            else:
                zf, th = o9_cpr(u, M, cfg.cpr_window)
                info["cpr"] = th
                _, lab = nearest(zf, M)
        z[k0:k0 + Fs] = zf
        dec[k0:k0 + Fs] = lab
        bi = int(round(math.log2(M))) - 2
        counts["sym"][bi] += Fs
        counts["bits"][bi] += Fs * (bi + 2)
        if ref is not None:
            r = np.asarray(ref[k0:k0 + Fs]).astype(np.int64)
            frame_err[fi] = (int(np.sum(lab != r)), int(np.sum(popcount(lab ^ r))))
            counts["sym_err"][bi] += frame_err[fi, 0]
            counts["bit_err"][bi] += frame_err[fi, 1]
        if keep:
            infos.append(info)
    out = dict(z=z, dec=dec, counts=counts, A=A, K=K, L=L, frame_err=frame_err, first=first, n=n,
               seq_state=seq_state)
    if keep:
        out.update(E=E, E0=e0, y=y, m0=m0, a=a, phi=phi, b=b, frames=infos, w_cd=w_cd, h=h)
    return out


def o11_q(counts: dict, fmt_index: Optional[int] = None) -> float:
    from .theory import q_from_ber
    be = counts["bit_err"] if fmt_index is None else counts["bit_err"][fmt_index]
    bt = counts["bits"] if fmt_index is None else counts["bits"][fmt_index]
    return q_from_ber(float(np.sum(be)) / float(np.sum(bt)))
