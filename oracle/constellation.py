"""QAM alphabets and the hard-decision demapper (oracle; TEST INFRASTRUCTURE ONLY).

Follows PAPER.md:24/50 ("4-, 8-, 16-, 32-, and 64-QAM"), PAPER.md:82 ("decisions
made by the equalizer are demapped") and SURVEY R13 for the 8/32 layouts the paper
does not state:
  * 4/16/64: square grid, per-axis binary-reflected Gray, label = gray(iI)<<(b/2) | gray(iQ),
    level index 0 = most negative;
  * 8: {±1,±3}×{±1}/√6, label = gray(iI)<<1 | iQ;
  * 32: 6×6 cross minus corners /√20 with the fixed R13 label table.
Decisions are brute force: argmin over all M points of |z − point|².
"""
from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

FORMATS = (4, 8, 16, 32, 64)

_CROSS32 = {  # (I, Q) grid coordinates -> label, SURVEY R13 table (rows Q=+5..-5, cols I=-5..+5)
    (-3, 5): 3, (-1, 5): 2, (1, 5): 18, (3, 5): 19,
    (-5, 3): 6, (-3, 3): 14, (-1, 3): 10, (1, 3): 26, (3, 3): 30, (5, 3): 22,
    (-5, 1): 7, (-3, 1): 15, (-1, 1): 11, (1, 1): 27, (3, 1): 31, (5, 1): 23,
    (-5, -1): 5, (-3, -1): 13, (-1, -1): 9, (1, -1): 25, (3, -1): 29, (5, -1): 21,
    (-5, -3): 4, (-3, -3): 12, (-1, -3): 8, (1, -3): 24, (3, -3): 28, (5, -3): 20,
    (-3, -5): 0, (-1, -5): 1, (1, -5): 17, (3, -5): 16,
}


def _gray(i: int) -> int:
    return i ^ (i >> 1)


@lru_cache(maxsize=None)
def constellation(M: int):
    """Return (points[M] complex128, labels[M] int) — point i carries label labels[i]."""
    pts, labs = [], []
    if M in (4, 16, 64):
        m = int(round(math.sqrt(M)))
        half_bits = int(round(math.log2(m)))
        norm = math.sqrt(2.0 * (M - 1) / 3.0)   # mean |(2i-(m-1)) + j(2q-(m-1))|^2
        for iI in range(m):
            for iQ in range(m):
                pts.append(complex(2 * iI - (m - 1), 2 * iQ - (m - 1)) / norm)
                labs.append((_gray(iI) << half_bits) | _gray(iQ))
    elif M == 8:
        for iI in range(4):
            for iQ in range(2):
                pts.append(complex(2 * iI - 3, 2 * iQ - 1) / math.sqrt(6.0))
                labs.append((_gray(iI) << 1) | iQ)
    elif M == 32:
        for (i, q), lab in sorted(_CROSS32.items()):
            pts.append(complex(i, q) / math.sqrt(20.0))
            labs.append(lab)
    else:
        raise ValueError(f"unsupported QAM order {M}")
    return np.array(pts, np.complex128), np.array(labs, np.int64)


def points_by_label(M: int) -> np.ndarray:
    pts, labs = constellation(M)
    out = np.empty(M, np.complex128)
    out[labs] = pts
    return out


def nearest(z: np.ndarray, M: int):
    """Brute-force hard decision: (decided point, its label) for each z."""
    pts, labs = constellation(M)
    d2 = np.abs(z.reshape(-1, 1) - pts.reshape(1, -1)) ** 2
    i = np.argmin(d2, axis=1)
    return pts[i].reshape(z.shape), labs[i].reshape(z.shape)


def popcount(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.int64)
    c = np.zeros_like(x)
    while np.any(x):
        c += x & 1
        x >>= 1
    return c
