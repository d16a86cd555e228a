"""GPU parity for the K3 configurations and failure semantics the first suite left out (VERDICT r01 "What's
missing" 4, "What's weak" 8): CPR under a real phase rotation (SURVEY P12(iv) bounded wander, P12(v) the
physical differential laser phase noise), the silent-frame / LS fallback (§8(b) errors: bad frame, z = 0,
decisions D(0)), every CPR window (256…4096, R12), and the short equalizers L = 3 and L = 5 (K3 templates
K = 1, 2). Same bar as test_gpu_parity: field / MF / EQ within 1e-4 (EQ frames over it must be proven
boundary flips), decisions ≥ 99.99 % identical, counts bit-exact where noiseless."""
import numpy as np
import pytest
import torch

from gpu_case import (F, eq_check, field_rel_err, make_case, make_silent_case, receiver_for, rel, run_gpu,
                      run_oracle)

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import constellation as C  # noqa: E402


def _evm_db(z, M):
    d, _ = C.nearest(z, M)
    return 10 * np.log10(np.mean(np.abs(z - d) ** 2))


def _parity(case, gpu, orc, dec_min=0.9999):
    assert field_rel_err(gpu, orc) <= 1e-4
    assert gpu["m0"] == orc["m0"] and rel(gpu["y"], orc["y"]) <= 1e-4
    ze, proven, _ = eq_check(gpu["z"], orc, case["ocfg"])
    agree = np.mean(gpu["dec"] == orc["dec"])
    assert agree >= dec_min, agree
    return ze, proven


# ----------------------------------------------------------------------------- CPR under rotation (P12)
@pytest.mark.parametrize("M,wander", [(4, 0.4), (16, 0.15), (64, 0.05)])
def test_cpr_phase_wander_parity(M, wander):
    """P12(iv): data-vs-tone phase wander A·sin(2π·50 kHz·t), amplitude ≤ 0.8× the R12 limit for M (4-QAM
    0.4 rad, 16-QAM 0.15, 64-QAM 0.05): each 256-symbol window rotates by up to A — the GPU's CPR must
    follow the oracle's and remove it (noiseless: zero errors; the residual is the rotation within a window)."""
    case = make_case(M=M, dl=32000.0, cspr=16.0, n=8 * F, seed=120 + M, wander_rad=wander)
    gpu, orc = run_gpu(case), run_oracle(case)
    _parity(case, gpu, orc, dec_min=1.0)
    assert gpu["stats"]["bit_err"] == [0] * 5 == list(orc["counts"]["bit_err"])
    assert abs(_evm_db(gpu["z"], M) - _evm_db(orc["z"], M)) < 0.05      # oracle: −39 / −47 / −52 dB
    # the rotation is real: the per-window CPR angles of the oracle span most of ±A
    th = np.concatenate([f["cpr"] for f in orc["frames"]])
    assert np.ptp(th) > wander


def test_cpr_phase_wander_noisy_q_parity():
    case = make_case(M=16, dl=112000.0, cspr=12.0, esn0=17.0, n=1 << 19, seed=131, wander_rad=0.1)
    gpu, orc = run_gpu(case), run_oracle(case)
    _parity(case, gpu, orc)
    from oracle import theory
    bits = sum(gpu["stats"]["bits"])
    bg, bo = sum(gpu["stats"]["bit_err"]), int(orc["counts"]["bit_err"].sum())
    assert bg > 100 and abs(theory.q_from_ber(bg / bits) - theory.q_from_ber(bo / bits)) <= 0.05


@pytest.mark.parametrize("M", [4, 16, 64])
def test_cpr_laser_phase_noise_parity(M):
    """P12(v): physical differential laser phase noise φ(t − τ) − φ(t), 100 kHz ECL, τ = 0.83 ns
    (10,000 km): too fast for any window — the CPR must not degrade EVM (oracle: −33.7 dB with W = 256 and
    with W = 4096), and the GPU must match the oracle."""
    case = make_case(M=M, dl=200000.0, cspr=16.0, n=4 * F, seed=140 + M, linewidth_hz=100e3)
    gpu, orc = run_gpu(case), run_oracle(case)
    _parity(case, gpu, orc)
    assert abs(_evm_db(gpu["z"], M) - _evm_db(orc["z"], M)) < 0.05


# ----------------------------------------------------------------------------- silent frames: the fallback path
def test_silent_frames_bad_fallback():
    """Frames with the tone but no modulation (float input I = I_ref): the MF output is exactly zero, the AGC
    power is zero — the frame cannot be trained. Both sides count it in bad_frames, output z = 0 and decide
    D(0) (ties to the lower level, R15); every other frame keeps parity. The two frames at the edges of the
    quiet stretch have an MF output that is exactly zero over most of the frame on the GPU and fftconvolve's
    rounding (~1e-16) in the oracle: their decisions there are not unique and are not compared."""
    case = make_silent_case()
    rx = receiver_for(case, keep=True, input_float=True)
    gpu, orc = run_gpu(case, rx=rx), run_oracle(case)
    s, c = gpu["stats"], orc["counts"]
    assert s["bad_frames"] == c["bad_frames"] == len(case["silent_frames"]) == 3
    assert s["dead_frames"] == 0 == c["dead_frames"]
    assert field_rel_err(gpu, orc) <= 1e-4 and rel(gpu["y"], orc["y"]) <= 1e-4
    zg, zo = gpu["z"].reshape(-1, 4096), orc["z"].reshape(-1, 4096)
    dg, do = gpu["dec"].reshape(-1, 4096), orc["dec"].reshape(-1, 4096)
    for fi in case["silent_frames"]:
        assert np.all(zg[fi] == 0) and np.all(zo[fi] == 0)
        assert np.array_equal(dg[fi], do[fi])
        assert np.all(dg[fi] == dg[fi][0])                       # one label: D(0)
    keep = [fi for fi in range(zg.shape[0]) if fi not in case["edge_frames"]]
    zmask = zg.copy()
    zmask[case["edge_frames"]] = zo[case["edge_frames"]]
    eq_check(zmask.reshape(-1), orc, case["ocfg"])
    # frames inside the quiet stretch that still carry power (its first and last frame: the neighbour's
    # carrier offset leaks through the MF) are decided on noise-free junk — every decision that differs must
    # sit at a slicer boundary (the oracle's z within 1e-3 of it); all other frames at the usual bar
    from gpu_case import _near_boundary
    quiet = [fi for fi in keep if fi in (case["silent_frames"][0] - 2, case["silent_frames"][-1] + 2)]
    normal = [fi for fi in keep if fi not in quiet]
    assert np.mean(dg[normal] == do[normal]) >= 0.9999
    for fi in quiet:
        bad_idx = np.nonzero(dg[fi] != do[fi])[0]
        near = {k for k, _, _ in _near_boundary(zo[fi][bad_idx], 16, 1e-3)}
        assert near == set(range(len(bad_idx))), (fi, len(bad_idx), len(near))
    se_g = s["sym_err"]
    assert sum(se_g) > 0                                          # silent frames do count as errors


# ----------------------------------------------------------------------------- CPR windows, short equalizers
@pytest.mark.parametrize("W", [512, 2048, 4096])
def test_cpr_window_parity(W):
    case = make_case(M=16, dl=112000.0, cspr=12.0, esn0=18.0, n=8 * F, seed=170, cpr_window=W, wander_rad=0.05)
    gpu, orc = run_gpu(case), run_oracle(case)
    _parity(case, gpu, orc)
    th = np.concatenate([f["cpr"] for f in orc["frames"]])
    assert len(th) == 8 * 4096 // W


@pytest.mark.parametrize("L,M,dl", [(3, 16, 0.0), (5, 64, 0.0), (5, 16, 8000.0), (3, 4, 4000.0)])
def test_short_equalizer_parity(L, M, dl):
    """eq_taps 3 and 5 instantiate K3<1> and K3<2> (rule-sized links need L ≥ 7)."""
    case = make_case(M=M, dl=dl, cspr=14.0, esn0=None, n=4 * F, seed=180 + L, eq_taps=L)
    rx = receiver_for(case, keep=True)
    assert rx.taps == L
    gpu, orc = run_gpu(case, rx=rx), run_oracle(case)
    assert orc["L"] == L
    _parity(case, gpu, orc, dec_min=1.0)
    assert gpu["stats"]["bit_err"] == [0] * 5 == list(orc["counts"]["bit_err"])


@pytest.mark.parametrize("L", [3, 5])
def test_short_equalizer_noisy_parity(L):
    case = make_case(M=16, dl=0.0, cspr=12.0, esn0=16.0, n=8 * F, seed=190 + L, eq_taps=L)
    gpu, orc = run_gpu(case), run_oracle(case)
    _parity(case, gpu, orc)


# ----------------------------------------------------------------------------- static CD + short block LS (NEXT-2)
@pytest.mark.parametrize("kw", [dict(M=4, dl=200000.0, esn0=12.0), dict(M=16, dl=112000.0, esn0=None),
                                dict(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, esn0=24.0),
                                dict(M=64, dl=32000.0, esn0=26.0, eq_taps=7)])
def test_static_cd_short_fir_parity(kw):
    """K2 with the complex RRC × CD-inverse filter (as in the DDLMS arrangement) feeding the block-LS K3 with
    L = 5 (θ₀ = centre spike), against the oracle's same arrangement."""
    case = make_case(cspr=12.0, n=8 * F, seed=211, static_cd=True, **kw)
    rx = receiver_for(case, keep=True)
    assert rx.taps == (kw.get("eq_taps") or 5)
    gpu, orc = run_gpu(case, rx=rx), run_oracle(case)
    _parity(case, gpu, orc, dec_min=1.0 if kw.get("esn0") is None else 0.9999)
    if kw.get("esn0") is None:
        assert gpu["stats"]["bit_err"] == [0] * 5 == list(orc["counts"]["bit_err"])
