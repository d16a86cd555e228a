"""oracle — plain fp64 CPU implementation of the KK receive chain (TEST INFRASTRUCTURE ONLY).

This package is the parity oracle for the CUDA path in `paper_2104_06311_b200/`.
It is written from the paper (§2 "DSP chain") and the readings of
SURVEY.md §8(c) (listed again in DESIGN.md), step by step in the paper's order,
with numpy/scipy library primitives as single steps and no blocking or fusion.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it. The product path never does, and the
oracle never imports the product package: the two share no code. The only shared
module is `kkgen` (seeded input generation; none of the method's arithmetic).

Parity status per function (pins in tests/test_oracle_*.py):
  constellation.*      pinned (P2: energy, bijection, Gray, map∘demap; P11 theory)
  theory.q_from_ber    pinned (P1: closed form / printed values)
  theory.ber_*         pinned (textbook QPSK/BPSK special cases + Monte-Carlo slicer)
  receiver.o1..o4      pinned (P3 exp-construction, P4 high-CSPR KK, P5 Hilbert pins)
  receiver.o5..o6      pinned (P7 mixer periodicity / tone-to-DC, carrier mean)
  receiver.o7          pinned (P6 brute-force convolution)
  receiver.cd_init     pinned (P8 fit error vs closed form C(nu))
  receiver.o8          pinned (P9 lstsq, P9b widely-linear, P10 noiseless BER 0, P11 AWGN Q)
  receiver.o9          pinned (P12 rotation recovery)
  receiver.o10/o11     pinned (P10/P11 counts; P1)
"""
from . import constellation, theory, receiver  # noqa: F401
from .receiver import OracleConfig, receive  # noqa: F401
