"""GPU parity for 2× KK upsampling (K1U; DESIGN.md §3 "KK upsampling") against the
fp64 oracle's O3u on identical seeded inputs. Same tolerances as tests/test_gpu_parity.py: field, MF and
equalizer output within 1e-4 relative, decisions ≥ 99.99 % identical, Q within 0.05 dB, noiseless counts
exact."""
import numpy as np
import pytest
import torch

from gpu_case import F, eq_check, field_rel_err, make_case, rel, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import theory  # noqa: E402


def _check(case, gpu, orc, dec_min=0.9999):
    fe = field_rel_err(gpu, orc)
    assert fe <= 1e-4, f"field rel err {fe:.3e}"
    ye = rel(gpu["y"], orc["y"])
    assert ye <= 1e-4, f"MF rel err {ye:.3e}"
    ze, _, _ = eq_check(gpu["z"], orc, case["ocfg"])
    agree = np.mean(gpu["dec"] == orc["dec"])
    assert agree >= dec_min, f"decision agreement {agree}"
    return fe, ye, ze


def test_up_halo_is_16656():
    case = make_case(M=4, n=F, upsample=2)
    assert case["halo"] == 16656
    gpu = run_gpu(case)
    assert gpu["rx"].halo == 16656


def test_up_noiseless_parity_and_exact_counts():
    case = make_case(M=16, cspr=8.0, n=1 << 16, seed=111, upsample=2)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check(case, gpu, orc, dec_min=1.0)
    s, c = gpu["stats"], orc["counts"]
    assert s["bit_err"] == list(c["bit_err"]) == [0] * 5 and s["sym"] == list(c["sym"])
    assert s["clamped"] == c["clamped"] and s["bad_frames"] == 0


@pytest.mark.parametrize("M,dl,cspr,esn0,noise", [
    (4, 200000.0, 10.0, 12.0, "white"),
    (64, 32000.0, 8.0, 26.0, "analytic"),
    (16, 112000.0, 6.0, 18.0, "white"),
    (32, 0.0, 12.0, 22.0, "analytic"),
])
def test_up_awgn_parity(M, dl, cspr, esn0, noise):
    case = make_case(M=M, dl=dl, cspr=cspr, esn0=esn0, noise=noise, n=1 << 17, seed=112, upsample=2)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check(case, gpu, orc)
    bits = sum(gpu["stats"]["bits"])
    be_g, be_o = sum(gpu["stats"]["bit_err"]), int(orc["counts"]["bit_err"].sum())
    if be_o > 20:
        assert abs(theory.q_from_ber(be_g / bits) - theory.q_from_ber(be_o / bits)) <= 0.05


def test_up_mixed_formats_ddlms_lower_sideband():
    case = make_case(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, cspr=10.0, esn0=24.0,
                     n=5 * F, seed=113, sideband=-1, upsample=2, eq_mode="ddlms")
    gpu, orc = run_gpu(case), run_oracle(case)
    _check(case, gpu, orc)


def test_up_chunk_invariance():
    case = make_case(M=16, dl=50000.0, cspr=8.0, esn0=20.0, n=4 * F, seed=114, upsample=2)
    whole = run_gpu(case, keep=False)
    parts = run_gpu(case, keep=False, chunk=F)
    assert np.array_equal(whole["dec"], parts["dec"])
    assert whole["stats"] == parts["stats"]


def test_up_float_input():
    case = make_case(M=16, dl=8000.0, cspr=8.0, esn0=22.0, n=2 * F, seed=115, upsample=2)
    orc = run_oracle(case)
    from paper_2104_06311_b200 import KK_STAGE_FIELD
    from gpu_case import receiver_for
    rx = receiver_for(case, keep=True, input_float=True)
    codes = case["codes"].to(torch.float32).cuda()
    dec = torch.zeros(case["n"] // 4, dtype=torch.uint8, device="cuda")
    rx.process(codes, case["first"], case["n"], decisions=dec)
    e0, E = rx.intermediate(KK_STAGE_FIELD)
    gpu = dict(E0=e0, E=E.cpu().numpy().astype(np.complex128))
    assert field_rel_err(gpu, orc) <= 1e-4
    assert np.mean(dec.cpu().numpy() == orc["dec"]) >= 0.9999
    rx.close()
