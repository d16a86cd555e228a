"""GPU parity on the nonlinear channel workload (kkgen/ssfm.py): codes propagated on
the GPU through 16 spans with SPM + ASE, received by the CUDA path over the whole 125-frame block, and by the
fp64 oracle on two frames of the same codes — decisions ≥ 99.99 % identical, equalizer output per frame
(gpu_case.eq_check)."""
import numpy as np
import pytest
import torch

from gpu_case import eq_check

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

import kkgen  # noqa: E402
from kkgen import ssfm  # noqa: E402
from oracle import receiver as R  # noqa: E402
from paper_2104_06311_b200 import KK_STAGE_EQ, Receiver  # noqa: E402

F = 16384


def test_ssfm_workload_parity():
    M = 64
    cfg = kkgen.LinkConfig(formats=(M,), cspr_db=8.0, seed=21)
    H = 16640
    w = ssfm.workload(cfg, ssfm.FiberLink(), ssfm.BLOCK, -4.0, H, n_spans=16, device="cuda")
    rx = Receiver(adc_scale=w["adc_scale"], ref_intensity=w["i_ref"], dispersion_ps_per_nm=w["dl_ps_nm"],
                  formats=(M,), max_samples_per_call=ssfm.BLOCK, keep_intermediate=True)
    dec = torch.zeros(ssfm.BLOCK // 4, dtype=torch.uint8, device="cuda")
    rx.process(w["codes"], 0, ssfm.BLOCK, ref=w["labels"].contiguous(), decisions=dec)
    z = rx.intermediate(KK_STAGE_EQ)[1].cpu().numpy().astype(np.complex128)
    st = rx.stats()
    rx.close()
    assert st["frames"] == 125 and st["bad_frames"] == 0
    ber = sum(st["bit_err"]) / sum(st["bits"])
    assert ber < 1e-2                                          # 64-QAM at 1600 km, -4 dBm: ~1e-3
    first, n = 60 * F, 2 * F
    codes = w["codes"][first:first + n + 2 * H].cpu().numpy()   # codes[0] is global sample -H
    ocfg = R.OracleConfig(formats=(M,), dispersion_ps_per_nm=w["dl_ps_nm"], adc_scale=w["adc_scale"],
                          ref_intensity=w["i_ref"])
    out = R.receive(codes, first, n, ocfg, ref=w["labels"][first // 4:(first + n) // 4].cpu().numpy())
    d = dec[first // 4:(first + n) // 4].cpu().numpy()
    assert np.mean(d == out["dec"]) >= 0.9999
    eq_check(z[first // 4:(first + n) // 4], out, ocfg)
