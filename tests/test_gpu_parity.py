"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical seeded int16 inputs.

Tolerances (BASELINE.json north_star): reconstructed field within 1e-4 relative RMS (relative to
the signal part E − A_f), MF output within 1e-4, equalizer output within 1e-4, decided symbols ≥ 99.99 %
identical, Q within 0.05 dB, error counts bit-exact in the noiseless case.
"""
import math

import numpy as np
import pytest
import torch

from gpu_case import F, HALO, eq_check, field_rel_err, make_case, rel, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_06311_b200 as P  # noqa: E402
from oracle import theory  # noqa: E402


def _check_all(case, gpu, orc, dec_min=0.9999, z_tol=1e-4):
    fe = field_rel_err(gpu, orc)
    assert fe <= 1e-4, f"field rel err {fe:.3e}"
    assert gpu["m0"] == orc["m0"]
    ye = rel(gpu["y"], orc["y"])
    assert ye <= 1e-4, f"MF rel err {ye:.3e}"
    ze, _, _ = eq_check(gpu["z"], orc, case["ocfg"], tol=z_tol)
    agree = np.mean(gpu["dec"] == orc["dec"])
    assert agree >= dec_min, f"decision agreement {agree}"
    return fe, ye, ze, agree


# ----------------------------------------------------------------------------- C1 (BASELINE configs[0])
def test_c1_b2b_noiseless_parity_and_exact_counts():
    case = make_case(M=4, n=1 << 16, seed=101)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc, dec_min=1.0)
    s, c = gpu["stats"], orc["counts"]
    assert s["sym_err"] == list(c["sym_err"]) and s["bit_err"] == list(c["bit_err"]) == [0] * 5
    assert s["bits"] == list(c["bits"]) and s["sym"] == list(c["sym"])
    assert s["frames"] == 4 and s["clamped"] == c["clamped"] and s["dead_frames"] == 0 and s["bad_frames"] == 0


@pytest.mark.parametrize("esn0,noise", [(8.0, "white"), (10.0, "white"), (12.0, "white"), (5.0, "analytic"),
                                        (7.0, "analytic")])
def test_c1_awgn_parity(esn0, noise):
    case = make_case(M=4, n=1 << 18, esn0=esn0, noise=noise, seed=102)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc)
    be_g, be_o = sum(gpu["stats"]["bit_err"]), int(orc["counts"]["bit_err"].sum())
    bits = sum(gpu["stats"]["bits"])
    assert abs(theory.q_from_ber(be_g / bits) - theory.q_from_ber(be_o / bits)) <= 0.05


# ----------------------------------------------------------------------------- every format, CD, noise
@pytest.mark.parametrize("M,dl,cspr,esn0", [
    (8, 0.0, 12.0, None), (16, 112000.0, 12.0, None), (32, 200000.0, 12.0, None), (64, 32000.0, 12.0, None),
    (4, 200000.0, 12.0, None), (16, 112000.0, 6.0, 17.0 + 10 * math.log10(12.5) - 10 * math.log10(1 + 10 ** 0.6)),
    (64, 32000.0, 12.0, 26.0), (32, 32000.0, 14.0, 22.0), (8, 200000.0, 10.0, 16.0)])
def test_format_parity(M, dl, cspr, esn0):
    case = make_case(M=M, dl=dl, cspr=cspr, esn0=esn0, n=1 << 17, seed=200 + M)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc, dec_min=1.0 if esn0 is None else 0.9999)
    if esn0 is None:
        assert gpu["stats"]["bit_err"] == [0] * 5 == list(orc["counts"]["bit_err"])
    else:
        bits = sum(gpu["stats"]["bits"])
        bg, bo = sum(gpu["stats"]["bit_err"]), int(orc["counts"]["bit_err"].sum())
        if 0 < bg and 0 < bo:
            assert abs(theory.q_from_ber(bg / bits) - theory.q_from_ber(bo / bits)) <= 0.05


def test_q_parity_large_64qam():
    case = make_case(M=64, dl=32000.0, cspr=12.0, esn0=24.0, n=1 << 20, seed=301)
    gpu, orc = run_gpu(case), run_oracle(case, keep=True)
    _check_all(case, gpu, orc)
    bits = sum(gpu["stats"]["bits"])
    qg = theory.q_from_ber(sum(gpu["stats"]["bit_err"]) / bits)
    qo = theory.q_from_ber(int(orc["counts"]["bit_err"].sum()) / bits)
    assert abs(qg - qo) <= 0.05


# ----------------------------------------------------------------------------- mixed formats (C5 shape)
def test_mixed_format_schedule():
    case = make_case(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, cspr=12.0, esn0=26.0,
                     n=10 * F, seed=501)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc)
    s, c = gpu["stats"], orc["counts"]
    assert s["sym"] == list(c["sym"]) and s["bits"] == list(c["bits"])
    assert all(v == 2 * 4096 for v in s["sym"])


# ----------------------------------------------------------------------------- KK exactness on GPU (P3 analogue)
def test_exp_construction_float_input():
    from paper_2104_06311_b200 import KK_STAGE_FIELD, Receiver
    rng = np.random.default_rng(1)
    N, first, n = 1024, 3 * F, 2 * F
    q = np.arange(3, 262)
    c = rng.standard_normal(len(q)) + 1j * rng.standard_normal(len(q))
    gidx = np.arange(first - HALO, first + n + HALO)
    z = (c[None, :] * np.exp(2j * np.pi * np.outer(gidx % N, q) / N)).sum(axis=1)
    z *= 0.6 / np.max(np.abs(z))
    E = 2.0 * np.exp(z)
    I = torch.tensor(np.abs(E) ** 2, dtype=torch.float32, device="cuda")
    rx = Receiver(adc_scale=1.0, ref_intensity=4.0, input_float=True, max_samples_per_call=n, keep_intermediate=True)
    rx.process(I, first, n)
    e0, Eg = rx.intermediate(KK_STAGE_FIELD)
    Et = E[HALO - F: HALO + n + F]
    assert e0 == first - F
    err = np.linalg.norm(Eg.cpu().numpy() - Et) / np.linalg.norm(Et)
    assert err <= 1e-5, err


# ----------------------------------------------------------------------------- determinism / sharding (P13)
def test_chunk_and_shard_invariance():
    case = make_case(M=16, dl=112000.0, cspr=10.0, esn0=16.0, n=8 * F, seed=13)
    whole = run_gpu(case, keep=True)
    chunked = run_gpu(case, keep=True, chunk=2 * F)
    assert np.array_equal(whole["dec"], chunked["dec"])
    assert np.array_equal(whole["z"], chunked["z"])                 # bit-identical
    for k in ("sym", "sym_err", "bits", "bit_err", "clamped", "frames"):
        assert whole["stats"][k] == chunked["stats"][k]
    # two "ranks": separate contexts on the two halves of the stream
    from paper_2104_06311_b200 import Receiver
    o = case["ocfg"]
    codes = case["codes"].cuda()
    decs = []
    for r in range(2):
        rx = Receiver(adc_scale=o.adc_scale, ref_intensity=o.ref_intensity, dispersion_ps_per_nm=case["dl"],
                      formats=case["formats"], max_samples_per_call=4 * F)
        d = torch.zeros(4 * 4096, dtype=torch.uint8, device="cuda")
        rx.process(codes, case["first"] + r * 4 * F, 4 * F, decisions=d, offset=r * 4 * F)
        decs.append(d.cpu().numpy())
    assert np.array_equal(np.concatenate(decs), whole["dec"])


def test_decision_paths_agree():
    """K3's decision phase has a specialised loop for the common case (square/rectangular format, labels staged
    by TMA, no z output) next to the general one (32-cross frames, z output, dead frames): both must give the
    same decisions and counters — run once without and once with the z output on a mixed 4…64-QAM stream."""
    case = make_case(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, cspr=10.0, esn0=15.0, n=10 * F,
                     seed=17)
    fast = run_gpu(case, keep=False)
    general = run_gpu(case, keep=True)
    assert np.array_equal(fast["dec"], general["dec"])
    for k in ("sym", "sym_err", "bits", "bit_err", "clamped", "frames", "bad_frames"):
        assert fast["stats"][k] == general["stats"][k], k
    assert sum(fast["stats"]["sym_err"]) > 0


@pytest.mark.parametrize("dl", [32000.0, 200000.0])    # K = 4 (double-buffered labels) and K = 7 (single buffer)
def test_unaligned_reference_labels(dl):
    """K3 stages the reference labels by TMA only from a 16-B-aligned buffer (kkrx.h: any alignment is
    accepted); a label buffer at an odd address takes the per-symbol load path. Decisions and every counter
    must equal the aligned run's, for both label-buffer layouts of K3 (two buffers for K ≤ 6, one for K = 7)."""
    from gpu_case import receiver_for
    case = make_case(formats=(4, 16, 64), segment_frames=1, dl=dl, cspr=10.0, esn0=15.0, n=6 * F, seed=23)
    n, first = case["n"], case["first"]
    codes = case["codes"].cuda()
    outs = []
    for off in (0, 1):
        buf = torch.zeros(n // 4 + 16, dtype=torch.uint8, device="cuda")
        ref = buf[off:off + n // 4]
        ref.copy_(case["ref"].cuda())
        assert (ref.data_ptr() % 16 == 0) == (off == 0)
        dec = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
        rx = receiver_for(case, keep=False)
        rx.process(codes, first, n, ref=ref, decisions=dec, offset=0)
        outs.append((dec.cpu().numpy(), rx.stats()))
        rx.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    for k in ("sym", "sym_err", "bits", "bit_err", "clamped", "frames", "bad_frames"):
        assert outs[0][1][k] == outs[1][1][k], k
    assert sum(outs[0][1]["sym_err"]) > 0


# ----------------------------------------------------------------------------- edge cases
def test_single_frame_and_stream_start():
    case = make_case(M=4, n=F, first=0, esn0=10.0, seed=5)        # first frame of the stream, n = one frame
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc)


def test_dead_frame():
    case = make_case(M=16, n=3 * F, seed=3)
    case["codes"] = case["codes"].clone()
    case["codes"][HALO + F: HALO + 2 * F] = 0
    gpu, orc = run_gpu(case), run_oracle(case)
    s = gpu["stats"]
    assert s["dead_frames"] == 1 == orc["counts"]["dead_frames"] and s["clamped"] == F
    assert np.array_equal(gpu["dec"], orc["dec"])
    assert np.all(gpu["z"][4096:8192] == 0)


def test_linear_only_and_cpr_windows():
    case = make_case(M=16, dl=32000.0, cspr=14.0, esn0=20.0, n=4 * F, seed=8, eq_widely_linear=False,
                     cpr_window=1024)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc)


def test_host_path_matches_device_path():
    case = make_case(M=16, dl=112000.0, cspr=10.0, esn0=16.0, n=8 * F, seed=21)
    dev = run_gpu(case, keep=False)
    from gpu_case import receiver_for
    rx = receiver_for(case, keep=False, max_samples=2 * F)        # forces 4 pipelined chunks
    codes = case["codes"].pin_memory()
    ref = case["ref"].pin_memory()
    dec = torch.zeros(case["n"] // 4, dtype=torch.uint8).pin_memory()
    rx.process_host(codes, case["first"], case["n"], ref=ref, decisions=dec)
    assert np.array_equal(dec.numpy().astype(np.int64), dev["dec"])
    s = rx.stats()
    for k in ("sym", "sym_err", "bits", "bit_err", "frames"):
        assert s[k] == dev["stats"][k]


def test_call_errors():
    case = make_case(M=4, n=2 * F, seed=1)
    from gpu_case import receiver_for
    rx = receiver_for(case, keep=False)
    codes = case["codes"].cuda()
    with pytest.raises(P.KKError) as e:
        rx.process(codes, case["first"] + 4, 2 * F)
    assert e.value.status == P.KK_ERR_ALIGN
    with pytest.raises(P.KKError) as e:
        rx.process(codes, case["first"], 4 * F)
    assert e.value.status == P.KK_ERR_CONFIG
    with pytest.raises(P.KKError) as e:
        P.kk_process_frames(rx.ctx, codes.data_ptr() + HALO * 2, case["first"], 100)
    assert e.value.status == P.KK_ERR_SHORT
    with pytest.raises(P.KKError) as e:
        P.kk_process_frames(rx.ctx, codes.data_ptr() + HALO * 2 + 2, case["first"], 2 * F)
    assert e.value.status == P.KK_ERR_ALIGN
    with pytest.raises(P.KKError) as e:
        P.kk_intermediate_range(rx.ctx, P.KK_STAGE_EQ)
    assert e.value.status == P.KK_ERR_STATE


# ----------------------------------------------------------------------------- paper arrangement (NEXT-1/2)
@pytest.mark.parametrize("M,dl,cspr,esn0", [(16, 0.0, 12.0, None), (16, 200000.0, 12.0, None),
                                            (64, 32000.0, 12.0, 26.0), (4, 200000.0, 12.0, 12.0),
                                            (32, 112000.0, 14.0, 22.0)])
def test_ddlms_mode_parity(M, dl, cspr, esn0):
    case = make_case(M=M, dl=dl, cspr=cspr, esn0=esn0, n=1 << 17, seed=600 + M, eq_mode="ddlms")
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc, dec_min=1.0 if esn0 is None else 0.9999)
    if esn0 is None:
        assert gpu["stats"]["bit_err"] == [0] * 5 == list(orc["counts"]["bit_err"])
    assert gpu["stats"]["sym"] == list(orc["counts"]["sym"])


def test_ddlms_mode_mixed_formats_and_chunking():
    case = make_case(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, cspr=12.0, esn0=26.0,
                     n=10 * F, seed=502, eq_mode="ddlms", ddlms_block=512, ddlms_warmup=768)
    whole = run_gpu(case)
    chunked = run_gpu(case, chunk=2 * F)
    orc = run_oracle(case)
    _check_all(case, whole, orc)
    assert np.array_equal(whole["dec"], chunked["dec"]) and np.array_equal(whole["z"], chunked["z"])


@pytest.mark.parametrize("eq_mode", ["block_ls", "ddlms"])
def test_lower_sideband(eq_mode):
    """σ = −1: data below the tone — φ and the LO mirror (R2), CD referenced to −f_c."""
    case = make_case(M=16, dl=112000.0, cspr=12.0, esn0=20.0, n=4 * F, seed=31, sideband=-1, eq_mode=eq_mode)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc)
    assert sum(gpu["stats"]["sym_err"]) < 0.05 * sum(gpu["stats"]["sym"])   # it actually demodulates


# ----------------------------------------------------------------------------- 8-bit ADC input, per-frame errors
def test_uint8_adc_input():
    """8-bit ADC codes (SPEC S:199's ADC width; KK_IN_UINT8): same parity bar on the same codes."""
    import dataclasses

    import kkgen
    from gpu_case import receiver_for
    from oracle import receiver as R
    case = make_case(M=16, dl=32000.0, cspr=12.0, esn0=18.0, n=4 * F, seed=41)
    lc = dataclasses.replace(case["lc"], adc_bits=8)
    g = kkgen.generate(lc, case["first"] - HALO, case["first"] + case["n"] + HALO)
    assert g["codes"].dtype == torch.uint8
    case8 = dict(case, codes=g["codes"], ocfg=R.OracleConfig(dispersion_ps_per_nm=case["dl"], adc_scale=lc.adc_scale,
                                                           ref_intensity=lc.i_ref, formats=case["formats"]))
    rx = receiver_for(case8, keep=True, input_uint8=True)
    gpu, orc = run_gpu(case8, rx=rx), run_oracle(case8)
    _check_all(case8, gpu, orc)


def test_adc_offset():
    """O1 with a nonzero ADC offset (kk_config.adc_offset: I = adc_scale·(code − adc_offset)): int16 codes
    shifted by −1000 with adc_offset = −1000 — the same parity bar against the oracle run on the shifted codes."""
    from gpu_case import receiver_for
    from oracle import receiver as R
    case = make_case(M=16, dl=32000.0, cspr=12.0, esn0=18.0, n=4 * F, seed=47)
    o = case["ocfg"]
    ocfg = R.OracleConfig(dispersion_ps_per_nm=case["dl"], adc_scale=o.adc_scale, ref_intensity=o.ref_intensity,
                          formats=case["formats"], adc_offset=-1000.0)
    case_o = dict(case, codes=(case["codes"].to(torch.int32) - 1000).to(torch.int16), ocfg=ocfg)
    rx = receiver_for(case_o, keep=True, adc_offset=-1000.0)
    gpu, orc = run_gpu(case_o, rx=rx), run_oracle(case_o)
    _check_all(case_o, gpu, orc)


def test_joint_intensity_scale():
    """The oracle's joint-scale covariance pin on the GPU: photocurrent (adc_scale) and I_ref both scaled by
    2^-80 ≈ 8e-25 — every clamp/silent threshold is relative to I_ref, so the fp32 path still meets the parity
    bar against the oracle of the scaled case (no frame turns silent, no sample clamps)."""
    from gpu_case import receiver_for
    from oracle import receiver as R
    c = 2.0 ** -80
    case = make_case(M=16, dl=32000.0, cspr=12.0, esn0=18.0, n=4 * F, seed=53)
    o = case["ocfg"]
    ocfg = R.OracleConfig(dispersion_ps_per_nm=case["dl"], adc_scale=o.adc_scale * c, ref_intensity=o.ref_intensity * c,
                          formats=case["formats"])
    case_s = dict(case, ocfg=ocfg)
    gpu, orc = run_gpu(case_s, rx=receiver_for(case_s, keep=True)), run_oracle(case_s)
    assert gpu["stats"]["bad_frames"] == 0 and orc["counts"]["bad_frames"] == 0
    _check_all(case_s, gpu, orc)


@pytest.mark.parametrize("eq_mode", ["block_ls", "ddlms"])
def test_per_frame_errors(eq_mode):
    case = make_case(M=64, dl=32000.0, cspr=12.0, esn0=22.0, n=6 * F, seed=43, eq_mode=eq_mode)
    from gpu_case import receiver_for
    rx = receiver_for(case, keep=False)
    codes, ref = case["codes"].cuda(), case["ref"].cuda()
    fe = torch.full((2 * 6,), -1, dtype=torch.int32, device="cuda")
    rx.process(codes, case["first"], case["n"], ref=ref, frame_errors=fe)
    st = rx.stats()
    fe = fe.cpu().numpy().reshape(-1, 2)
    assert fe[:, 1].sum() == sum(st["bit_err"]) and fe[:, 0].sum() == sum(st["sym_err"])
    orc = run_oracle(case, keep=False)
    agree = np.abs(fe - orc["frame_err"]).sum()
    assert agree <= max(2, 0.002 * orc["frame_err"].sum())
    from paper_2104_06311_b200 import qtrace
    bins = qtrace.bin_q(fe[:, 1], [4096 * 6] * 6, frames_per_bin=3)
    assert len(bins) == 2 and all(b["q_db"] is not None for b in bins)


@pytest.mark.parametrize("cspr", [4.0, 8.0, 12.0, 16.0])
def test_c2_cspr_sweep_q_parity(cspr):
    """BASELINE configs[1] sweep axis: 16-QAM, 5600 km, OSNR 17 dB, CSPR swept (Q within 0.05 dB)."""
    import kkgen
    case = make_case(M=16, dl=112000.0, cspr=cspr, esn0=kkgen.esn0_from_osnr(17.0, cspr), n=1 << 20, seed=201)
    gpu, orc = run_gpu(case, keep=False), run_oracle(case, keep=False)
    assert np.mean(gpu["dec"] == orc["dec"]) >= 0.9999
    bits = sum(gpu["stats"]["bits"])
    qg = theory.q_from_ber(sum(gpu["stats"]["bit_err"]) / bits)
    qo = theory.q_from_ber(int(orc["counts"]["bit_err"].sum()) / bits)
    assert abs(qg - qo) <= 0.05, (qg, qo)
    assert gpu["stats"]["clamped"] == orc["counts"]["clamped"]


# ----------------------------------------------------------------------------- minimum-phase violated
@pytest.mark.parametrize("M,cspr,esn0,up", [(16, 0.0, 18.0, 1), (4, 1.0, 12.0, 1), (16, 2.0, 18.0, 2),
                                            (64, 4.0, 26.0, 1)])
def test_very_low_cspr_parity(M, cspr, esn0, up):
    """CSPR 0–4 dB: the minimum-phase condition fails (SER 7–44 %) and intensities touch zero (clamped
    samples); the fp32 path must still track the fp64 oracle (measured: field 3e-7 … 1.6e-6, decisions 100 %)."""
    case = make_case(M=M, dl=32000.0, cspr=cspr, esn0=esn0, n=1 << 17, seed=141, upsample=up)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc)
    assert gpu["stats"]["clamped"] == orc["counts"]["clamped"]


# ----------------------------------------------------------------------------- MF grid 8192/7168
@pytest.mark.parametrize("kw", [dict(M=16, dl=112000.0, esn0=17.0), dict(M=64, dl=32000.0, esn0=26.0, upsample=2),
                                dict(M=16, dl=112000.0, esn0=18.0, eq_mode="ddlms"),
                                dict(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, esn0=24.0, sideband=-1)])
def test_mf8192_grid_parity(kw):
    """The FFT8192/hop-7168 overlap-save grid computes the same exact linear convolution as the 4096/3072 one
    (K2 template): MF output, equalizer output and decisions against the grid-independent oracle."""
    case = make_case(n=5 * F, first=3 * F, seed=151, **kw)
    from gpu_case import receiver_for
    rx = receiver_for(case, keep=True, mf_fft_n=8192)
    gpu, orc = run_gpu(case, rx=rx), run_oracle(case)
    _check_all(case, gpu, orc)


# ----------------------------------------------------------------------------- far into the stream
@pytest.mark.parametrize("kw", [dict(M=16, dl=112000.0, esn0=17.0),
                                dict(formats=(4, 8, 16, 32, 64), segment_frames=3, dl=32000.0, esn0=24.0,
                                     eq_mode="ddlms"),
                                dict(M=64, dl=32000.0, esn0=26.0, upsample=2)])
def test_global_index_2_40(kw):
    """first_sample = 2^40 (≈ 4.6 min of stream): the LO index (129·n mod 1000), frame and segment numbers,
    the format schedule and the generator's hash all run on 64-bit global positions."""
    case = make_case(n=3 * F, first=1 << 40, seed=161, **kw)
    gpu, orc = run_gpu(case), run_oracle(case)
    _check_all(case, gpu, orc)
