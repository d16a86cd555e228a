"""Closed-form Q(BER) and AWGN BER of the QAM alphabets (oracle; TEST INFRASTRUCTURE ONLY).

q_from_ber: Q = 20·log10(√2·erfcinv(2·BER)) ("Q-factors were
estimated from BER"). Undefined (ValueError) unless 0 < BER < 0.5.

ber_awgn: exact finite sums for the hard-decision slicer on circular complex AWGN with
E_s = 1: square QAM and the 8-QAM rectangle are separable, so per-axis PAM
interval probabilities weighted by the Gray-label Hamming distance give the BER exactly;
the 32-cross is integrated cell by cell (rectangular cells separable, the four corner
cells split on the diagonal by 1-D quadrature).
"""
from __future__ import annotations

import math

import numpy as np
from scipy import integrate, special

from .constellation import constellation


def q_from_ber(ber: float) -> float:
    if not (0.0 < ber < 0.5):
        raise ValueError("Q undefined unless 0 < BER < 0.5")
    return 20.0 * math.log10(math.sqrt(2.0) * special.erfcinv(2.0 * ber))


def _Phi(x):
    return 0.5 * special.erfc(-np.asarray(x, dtype=np.float64) / math.sqrt(2.0))


def _pam_transition(levels: np.ndarray, sigma: float) -> np.ndarray:
    """P[j | i] for a 1-D slicer with midpoint boundaries between sorted levels."""
    b = np.concatenate(([-np.inf], 0.5 * (levels[1:] + levels[:-1]), [np.inf]))
    P = _Phi((b[None, 1:] - levels[:, None]) / sigma) - _Phi((b[None, :-1] - levels[:, None]) / sigma)
    return P


def _hd(a: int, b: int) -> int:
    return bin(a ^ b).count("1")


def ber_awgn(M: int, esn0_db: float) -> float:
    """Exact BER of the (brute-force = per-axis) hard slicer, E_s = 1, complex AWGN N0 = 1/(Es/N0)."""
    n0 = 10.0 ** (-esn0_db / 10.0)
    sig = math.sqrt(n0 / 2.0)                         # per-axis std
    gray = lambda i: i ^ (i >> 1)
    if M in (4, 16, 64):
        m = int(round(math.sqrt(M)))
        lv = np.array([2 * i - (m - 1) for i in range(m)], float) / math.sqrt(2.0 * (M - 1) / 3.0)
        P = _pam_transition(lv, sig)
        e_axis = sum(P[i, j] * _hd(gray(i), gray(j)) for i in range(m) for j in range(m)) / m
        return 2.0 * e_axis / math.log2(M)
    if M == 8:
        lvI = np.array([-3, -1, 1, 3], float) / math.sqrt(6.0)
        lvQ = np.array([-1, 1], float) / math.sqrt(6.0)
        PI, PQ = _pam_transition(lvI, sig), _pam_transition(lvQ, sig)
        eI = sum(PI[i, j] * _hd(gray(i), gray(j)) for i in range(4) for j in range(4)) / 4
        eQ = sum(PQ[i, j] * (i != j) for i in range(2) for j in range(2)) / 2
        return (eI + eQ) / 3.0
    if M == 32:
        return _ber_cross32(sig)
    raise ValueError(M)


def _ber_cross32(sig: float) -> float:
    pts, labs = constellation(32)
    s = math.sqrt(20.0)
    grid = np.array([-5, -3, -1, 1, 3, 5], float)
    bnd = np.array([-np.inf, -4, -2, 0, 2, 4, np.inf])
    lab_of = {(int(round(p.real * s)), int(round(p.imag * s))): int(l) for p, l in zip(pts, labs)}
    total = 0.0
    for p, l in zip(pts, labs):
        px, py = p.real * s, p.imag * s                 # grid units; noise std sig*s per axis
        sg = sig * s
        PI = _Phi((bnd[1:] - px) / sg) - _Phi((bnd[:-1] - px) / sg)
        PQ = _Phi((bnd[1:] - py) / sg) - _Phi((bnd[:-1] - py) / sg)
        for a in range(6):
            for b in range(6):
                gx, gy = int(grid[a]), int(grid[b])
                if abs(gx) == 5 and abs(gy) == 5:       # corner cell: split on |y| = |x|
                    sx, sy = np.sign(gx), np.sign(gy)
                    # mass with |x| > |y| inside the cell -> (5sx, 3sy); else (3sx, 5sy)
                    f = lambda u: (math.exp(-0.5 * ((sx * u - px) / sg) ** 2) / (sg * math.sqrt(2 * math.pi))
                                   * float(abs(_Phi((sy * u - py) / sg) - _Phi((sy * 4 - py) / sg))))
                    m_x = integrate.quad(f, 4.0, np.inf, epsabs=1e-16, epsrel=1e-10, limit=200)[0]
                    m_all = PI[a] * PQ[b]
                    total += m_x * _hd(l, lab_of[(5 * int(sx), 3 * int(sy))])
                    total += (m_all - m_x) * _hd(l, lab_of[(3 * int(sx), 5 * int(sy))])
                else:
                    total += PI[a] * PQ[b] * _hd(l, lab_of[(gx, gy)])
    return total / 32.0 / 5.0
