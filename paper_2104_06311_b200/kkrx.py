"""ctypes binding of libkkrx.so (include/kkrx.h) — argument marshalling only.

Every function here has the name of the C entry point it calls; all arithmetic of the receive chain runs
in the library's CUDA kernels. Device buffers are passed as raw device addresses (torch.Tensor.data_ptr()),
streams as raw cudaStream_t handles (torch.cuda.Stream.cuda_stream). There is no CPU fallback: importing
this module fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_uint8, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KK_LIB", os.path.join(HERE, "libkkrx.so"))   # KK_LIB: A/B experiments only

KK_OK, KK_ERR_CONFIG, KK_ERR_ALIGN, KK_ERR_SHORT, KK_ERR_NULL = 0, -1, -2, -3, -4
KK_ERR_NOMEM, KK_ERR_CUDA, KK_ERR_DOMAIN, KK_ERR_STATE = -5, -6, -7, -8
KK_IN_INT16, KK_IN_FLOAT32, KK_IN_UINT8 = 0, 1, 2
KK_EQ_BLOCK_LS, KK_EQ_DDLMS = 0, 1
KK_STAGE_FIELD, KK_STAGE_MF, KK_STAGE_EQ = 0, 1, 2
KK_STATS_WORDS = 24
HALO = 16640


class kk_config(ctypes.Structure):
    _fields_ = [
        ("fs_hz", c_double), ("baud_hz", c_double),
        ("lo_num", c_int32), ("lo_den", c_int32), ("sideband", c_int32), ("rrc_span_sym", c_int32),
        ("rolloff", c_double),
        ("hilbert_n", c_int32), ("hilbert_hop", c_int32), ("mf_fft_n", c_int32), ("mf_hop", c_int32),
        ("frame_symbols", c_int32), ("eq_taps", c_int32), ("eq_widely_linear", c_int32), ("cpr_window", c_int32),
        ("eq_ridge", c_double), ("dispersion_ps_per_nm", c_double), ("lambda_m", c_double),
        ("input_dtype", c_int32), ("adc_scale", c_float), ("adc_offset", c_float), ("ref_intensity", c_float),
        ("clamp_rel", c_float),
        ("format_schedule", POINTER(c_uint8)), ("n_segments", c_int32), ("default_format", c_int32),
        ("segment_frames", c_int64), ("max_samples_per_call", c_int64), ("device", c_int32),
        ("keep_intermediate", c_int32),
        ("eq_mode", c_int32), ("ddlms_block", c_int32), ("ddlms_warmup", c_int32), ("debug_guard", c_int32),
        ("ddlms_mu_warm", c_double), ("ddlms_mu", c_double),
        ("upsample", c_int32), ("ref_prbs", c_int32), ("ref_seed", c_uint32), ("reserved2", c_int32),
        ("ddlms_mu_mid", c_double), ("static_cd", c_int32), ("reserved3", c_int32),
    ]


class kk_stats_t(ctypes.Structure):
    _fields_ = [("sym", c_uint64 * 5), ("sym_err", c_uint64 * 5), ("bits", c_uint64 * 5), ("bit_err", c_uint64 * 5),
                ("clamped", c_uint64), ("frames", c_uint64), ("dead_frames", c_uint64), ("bad_frames", c_uint64)]


class KKError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        super().__init__(f"{where}: {kk_strerror(status)} ({status}) {detail}".rstrip())
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libkkrx.so not built at {LIB_PATH}: run `python paper_2104_06311_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "kk_config_default": (None, [POINTER(kk_config)]),
        "kk_config_sizeof": (c_size_t, []),
        "kk_stats_sizeof": (c_size_t, []),
        "kk_init": (c_int, [POINTER(kk_config), POINTER(c_void_p)]),
        "kk_halo": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int64)]),
        "kk_eq_taps": (c_int, [c_void_p, POINTER(c_int32)]),
        "kk_process_frames": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
        "kk_process_frames_ex": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                         c_void_p]),
        "kk_process_frames_host": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
        "kk_stats": (c_int, [c_void_p, POINTER(kk_stats_t)]),
        "kk_stats_device": (c_int, [c_void_p, c_void_p, c_void_p]),
        "kk_reset_stats": (c_int, [c_void_p, c_void_p]),
        "kk_intermediate_range": (c_int, [c_void_p, c_int, POINTER(c_int64), POINTER(c_int64)]),
        "kk_get_intermediate": (c_int, [c_void_p, c_int, c_void_p, c_size_t, c_void_p]),
        "kk_enable_timing": (c_int, [c_void_p, c_int]),
        "kk_kernel_times": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int64), c_int]),
        "kk_q_from_ber": (c_int, [c_double, POINTER(c_double)]),
        "kk_check_guards": (c_int, [c_void_p, POINTER(c_int32)]),
        "kk_destroy": (None, [c_void_p]),
        "kk_strerror": (c_char_p, [c_int]),
        "kk_last_error": (c_char_p, [c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.kk_config_sizeof() != ctypes.sizeof(kk_config) or lib.kk_stats_sizeof() != ctypes.sizeof(kk_stats_t):
        raise ImportError("kk_config / kk_stats_t layout mismatch between libkkrx.so and the binding")
    return lib


lib = _load()


def _check(st: int, where: str, ctx=None):
    if st != KK_OK:
        detail = lib.kk_last_error(ctx).decode() if ctx else ""
        raise KKError(st, where, detail)


# ---------------------------------------------------------------- 1:1 wrappers
def kk_config_default() -> kk_config:
    c = kk_config()
    lib.kk_config_default(ctypes.byref(c))
    return c


def kk_init(cfg: kk_config) -> c_void_p:
    ctx = c_void_p()
    _check(lib.kk_init(ctypes.byref(cfg), ctypes.byref(ctx)), "kk_init")
    return ctx


def kk_halo(ctx):
    l, r = c_int64(), c_int64()
    _check(lib.kk_halo(ctx, ctypes.byref(l), ctypes.byref(r)), "kk_halo", ctx)
    return l.value, r.value


def kk_eq_taps(ctx) -> int:
    t = c_int32()
    _check(lib.kk_eq_taps(ctx, ctypes.byref(t)), "kk_eq_taps", ctx)
    return t.value


def kk_process_frames(ctx, d_adc: int, first_sample: int, n_samples: int, d_ref: int = 0, d_decisions: int = 0,
                      stream: int = 0):
    _check(lib.kk_process_frames(ctx, c_void_p(d_adc), first_sample, n_samples, c_void_p(d_ref or None),
                                 c_void_p(d_decisions or None), c_void_p(stream or None)), "kk_process_frames", ctx)


def kk_process_frames_ex(ctx, d_adc: int, first_sample: int, n_samples: int, d_ref: int = 0, d_decisions: int = 0,
                         d_frame_errors: int = 0, stream: int = 0):
    _check(lib.kk_process_frames_ex(ctx, c_void_p(d_adc), first_sample, n_samples, c_void_p(d_ref or None),
                                    c_void_p(d_decisions or None), c_void_p(d_frame_errors or None),
                                    c_void_p(stream or None)), "kk_process_frames_ex", ctx)


def kk_process_frames_host(ctx, h_adc: int, first_sample: int, n_samples: int, h_ref: int = 0, h_decisions: int = 0):
    _check(lib.kk_process_frames_host(ctx, c_void_p(h_adc), first_sample, n_samples, c_void_p(h_ref or None),
                                      c_void_p(h_decisions or None)), "kk_process_frames_host", ctx)


def kk_stats(ctx) -> dict:
    s = kk_stats_t()
    _check(lib.kk_stats(ctx, ctypes.byref(s)), "kk_stats", ctx)
    return dict(sym=list(s.sym), sym_err=list(s.sym_err), bits=list(s.bits), bit_err=list(s.bit_err),
                clamped=s.clamped, frames=s.frames, dead_frames=s.dead_frames, bad_frames=s.bad_frames)


def kk_stats_device(ctx, d_out: int, stream: int = 0):
    _check(lib.kk_stats_device(ctx, c_void_p(d_out), c_void_p(stream or None)), "kk_stats_device", ctx)


def kk_reset_stats(ctx, stream: int = 0):
    _check(lib.kk_reset_stats(ctx, c_void_p(stream or None)), "kk_reset_stats", ctx)


def kk_intermediate_range(ctx, stage: int):
    a, b = c_int64(), c_int64()
    _check(lib.kk_intermediate_range(ctx, stage, ctypes.byref(a), ctypes.byref(b)), "kk_intermediate_range", ctx)
    return a.value, b.value


def kk_get_intermediate(ctx, stage: int, d_dst: int, nbytes: int, stream: int = 0):
    _check(lib.kk_get_intermediate(ctx, stage, c_void_p(d_dst), nbytes, c_void_p(stream or None)),
           "kk_get_intermediate", ctx)


def kk_enable_timing(ctx, enable: bool = True):
    _check(lib.kk_enable_timing(ctx, int(enable)), "kk_enable_timing", ctx)


def kk_kernel_times(ctx, reset: bool = False):
    """([ms_K1, ms_K2, ms_K3], [launches_K1, launches_K2, launches_K3]) accumulated while timing was enabled."""
    ms, n = (c_double * 3)(), (c_int64 * 3)()
    _check(lib.kk_kernel_times(ctx, ms, n, int(reset)), "kk_kernel_times", ctx)
    return list(ms), list(n)


def kk_q_from_ber(ber: float) -> float:
    q = c_double()
    _check(lib.kk_q_from_ber(ber, ctypes.byref(q)), "kk_q_from_ber")
    return q.value


def kk_check_guards(ctx) -> int:
    """Number of canary-guarded buffers checked (0 unless debug_guard); raises KKError on a bounds violation."""
    n = c_int32()
    _check(lib.kk_check_guards(ctx, ctypes.byref(n)), "kk_check_guards", ctx)
    return n.value


def kk_destroy(ctx):
    lib.kk_destroy(ctx)


def kk_strerror(status: int) -> str:
    return lib.kk_strerror(status).decode()


def kk_last_error(ctx) -> str:
    return lib.kk_last_error(ctx).decode()


def stats_from_words(words) -> dict:
    """Decode the 24-word counter layout written by kk_stats_device (e.g. after an NCCL allreduce)."""
    w = [int(x) for x in words]
    return dict(sym=w[0:5], sym_err=w[5:10], bits=w[10:15], bit_err=w[15:20], clamped=w[20], frames=w[21],
                dead_frames=w[22], bad_frames=w[23])
