"""paper_2104_06311_b200 — B200 (sm_100a) Kramers-Kronig receive chain of arXiv 2104.06311.

The product is libkkrx.so (C ABI: include/kkrx.h; CUDA kernels in csrc/). `kkrx` is its ctypes binding
and `Receiver` a marshalling convenience. Importing fails loudly if the library is not built: there is
no CPU fallback.
"""
from .kkrx import *  # noqa: F401,F403
from .receiver import Receiver  # noqa: F401
