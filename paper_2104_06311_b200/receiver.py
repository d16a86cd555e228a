"""Receiver: a convenience holder around one libkkrx context (argument marshalling only).

It fills a kk_config from keyword arguments, keeps the context and passes torch tensors' device addresses
and the current CUDA stream to the C ABI. Every step of the chain runs in libkkrx's kernels.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import kkrx


class Receiver:
    def __init__(self, *, adc_scale: float, ref_intensity: float, adc_offset: float = 0.0,
                 dispersion_ps_per_nm: float = 0.0, formats: Sequence[int] = (4,), segment_frames: int = 1 << 30,
                 max_samples_per_call: int = 1 << 24, device: int = 0, keep_intermediate: bool = False,
                 eq_taps: int = 0, widely_linear: bool = True, cpr_window: int = 256, eq_ridge: float = 1e-3,
                 input_float: bool = False, input_uint8: bool = False, sideband: int = 1, lo_num: int = 129, lo_den: int = 1000,
                 clamp_rel: float = 1e-12, rolloff: float = 0.01, rrc_span_sym: int = 256,
                 eq_mode: str = "block_ls", ddlms_block: int = 512, ddlms_warmup: int = 1024,
                 ddlms_mu_warm: float = 2e-3, ddlms_mu: float = 2.5e-4, ddlms_mu_mid: float = 5e-4,
                 debug_guard: bool = False,
                 upsample: int = 1, mf_fft_n: int = 4096, ref_prbs_seed: Optional[int] = None,
                 ref_prbs_kind: str = "hash", static_cd: bool = False):
        cfg = kkrx.kk_config_default()
        cfg.adc_scale, cfg.adc_offset, cfg.ref_intensity = adc_scale, adc_offset, ref_intensity
        cfg.dispersion_ps_per_nm = dispersion_ps_per_nm
        cfg.max_samples_per_call = max_samples_per_call
        cfg.device = device
        cfg.keep_intermediate = int(keep_intermediate)
        cfg.eq_taps = eq_taps
        cfg.eq_widely_linear = int(widely_linear)
        cfg.cpr_window = cpr_window
        cfg.eq_ridge = eq_ridge
        cfg.input_dtype = (kkrx.KK_IN_FLOAT32 if input_float else kkrx.KK_IN_UINT8 if input_uint8
                           else kkrx.KK_IN_INT16)
        cfg.sideband, cfg.lo_num, cfg.lo_den = sideband, lo_num, lo_den
        cfg.clamp_rel, cfg.rolloff, cfg.rrc_span_sym = clamp_rel, rolloff, rrc_span_sym
        cfg.eq_mode = {"block_ls": kkrx.KK_EQ_BLOCK_LS, "ddlms": kkrx.KK_EQ_DDLMS}[eq_mode]
        cfg.ddlms_block, cfg.ddlms_warmup = ddlms_block, ddlms_warmup
        cfg.ddlms_mu_warm, cfg.ddlms_mu, cfg.ddlms_mu_mid = ddlms_mu_warm, ddlms_mu, ddlms_mu_mid
        cfg.debug_guard = int(debug_guard)
        cfg.static_cd = int(static_cd)
        cfg.upsample = upsample
        cfg.mf_fft_n, cfg.mf_hop = mf_fft_n, mf_fft_n - 1024      # MF overlap-save grid (4096/3072 or 8192/7168)
        if ref_prbs_seed is not None:                                # the transmitter's known labels, generated on the GPU
            cfg.ref_prbs = {"hash": 1, "prbs31": 2}[ref_prbs_kind]      # the synthetic hash | ITU-T PRBS-31
            cfg.ref_seed = ref_prbs_seed & 0xFFFFFFFF
        fm = list(formats)
        self._sched = (ctypes.c_uint8 * len(fm))(*fm)
        cfg.format_schedule = ctypes.cast(self._sched, ctypes.POINTER(ctypes.c_uint8))
        cfg.n_segments = len(fm)
        cfg.segment_frames = segment_frames
        cfg.default_format = fm[0]
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        self.input_dtype = torch.float32 if input_float else torch.uint8 if input_uint8 else torch.int16
        self.ctx = kkrx.kk_init(cfg)
        self.halo = kkrx.kk_halo(self.ctx)[0]
        self.taps = kkrx.kk_eq_taps(self.ctx)

    # ------------------------------------------------------------------ processing
    def process(self, adc: torch.Tensor, first_sample: int, n_samples: int, ref: Optional[torch.Tensor] = None,
                decisions: Optional[torch.Tensor] = None, offset: int = 0, stream: Optional[torch.cuda.Stream] = None,
                frame_errors: Optional[torch.Tensor] = None):
        """adc: device tensor; element `offset` is global sample first_sample − halo (so the core starts at
        offset + halo). ref / decisions: device uint8 tensors of n_samples/4 labels (nullable).
        frame_errors: optional device int32 tensor of 2·n_samples/16384 (symbol, bit errors per frame)."""
        assert adc.is_cuda and adc.dtype == self.input_dtype
        core = adc.data_ptr() + (offset + self.halo) * adc.element_size()
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        if frame_errors is not None:
            assert frame_errors.is_cuda and frame_errors.dtype == torch.int32
            assert frame_errors.numel() >= 2 * (n_samples // 16384)
            kkrx.kk_process_frames_ex(self.ctx, core, first_sample, n_samples,
                                      ref.data_ptr() if ref is not None else 0,
                                      decisions.data_ptr() if decisions is not None else 0,
                                      frame_errors.data_ptr(), s)
            return
        kkrx.kk_process_frames(self.ctx, core, first_sample, n_samples,
                               ref.data_ptr() if ref is not None else 0,
                               decisions.data_ptr() if decisions is not None else 0, s)

    def process_host(self, adc: torch.Tensor, first_sample: int, n_samples: int, ref: Optional[torch.Tensor] = None,
                     decisions: Optional[torch.Tensor] = None, offset: int = 0):
        """End-to-end path with HOST (pinned) tensors; same layout as process()."""
        assert not adc.is_cuda
        core = adc.data_ptr() + (offset + self.halo) * adc.element_size()
        kkrx.kk_process_frames_host(self.ctx, core, first_sample, n_samples,
                                    ref.data_ptr() if ref is not None else 0,
                                    decisions.data_ptr() if decisions is not None else 0)

    def stats(self) -> dict:
        return kkrx.kk_stats(self.ctx)

    def stats_device(self, out: torch.Tensor, stream: Optional[torch.cuda.Stream] = None):
        assert out.is_cuda and out.dtype in (torch.int64, torch.uint64) and out.numel() >= kkrx.KK_STATS_WORDS
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        kkrx.kk_stats_device(self.ctx, out.data_ptr(), s)

    def reset_stats(self, stream: Optional[torch.cuda.Stream] = None):
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        kkrx.kk_reset_stats(self.ctx, s)

    def intermediate(self, stage: int):
        """(first global index, complex64 device tensor) of the last call's FIELD / MF / EQ output."""
        first, count = kkrx.kk_intermediate_range(self.ctx, stage)
        out = torch.empty(count, dtype=torch.complex64, device=self.device)
        kkrx.kk_get_intermediate(self.ctx, stage, out.data_ptr(), count * 8,
                                 torch.cuda.current_stream(self.device).cuda_stream)
        return first, out

    def check_guards(self) -> int:
        """kk_check_guards: raises KKError if any kernel wrote outside its scratch buffer (debug_guard=True)."""
        return kkrx.kk_check_guards(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            kkrx.kk_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
