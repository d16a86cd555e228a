"""Binned Q-factor traces from per-frame error counts ("The short-term averaged Q-factors were
estimated from BER in bins of 21 ms"). Host-side bookkeeping only: the counts come from
kk_process_frames_ex, the BER→Q map from the library's kk_q_from_ber.

A 21 ms bin at 4 GS/s is 84·10⁶ samples = 5126.95 frames of 16,384 samples; bins here are whole frames
(`frames_per_bin`, default 5127 = 21.0 ms to within 0.001 %)."""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np

from . import kkrx

FRAME_SAMPLES = 16384
FS = 4e9
BIN_21MS_FRAMES = int(round(21e-3 * FS / FRAME_SAMPLES))    # 5127


def bin_q(frame_bit_errors: Sequence[int], bits_per_frame: Sequence[int], frames_per_bin: int = BIN_21MS_FRAMES):
    """Per bin: (start time s, bits, bit errors, BER, Q dB or None when BER ∉ (0, 0.5))."""
    be = np.asarray(frame_bit_errors, dtype=np.int64)
    bits = np.asarray(bits_per_frame, dtype=np.int64)
    out = []
    for b0 in range(0, len(be) - frames_per_bin + 1, frames_per_bin):
        e, n = int(be[b0:b0 + frames_per_bin].sum()), int(bits[b0:b0 + frames_per_bin].sum())
        ber = e / n
        q = kkrx.kk_q_from_ber(ber) if 0.0 < ber < 0.5 else None
        out.append(dict(t_s=b0 * FRAME_SAMPLES / FS, bits=n, bit_errors=e, ber=ber, q_db=q))
    return out
