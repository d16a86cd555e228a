"""GPU bounds checks (device sanitizers are not available on the GPU pool, so the library checks itself).

* Writes: every scratch buffer of the context sits between 64 KiB canaries (kk_config.debug_guard = 1) and
  kk_check_guards verifies them after the calls; the caller's own output buffers (decisions, per-frame
  errors) are embedded in sentinel-filled pads that must come back untouched.
* Reads: the input codes and reference labels are embedded in poisoned pads (NaN / full-scale codes /
  0xFF labels) just outside the [first − halo, first + n + halo) window the ABI says is read; any read
  past it changes the result, which must be bit-identical to an unpadded, unguarded run (the kernels are
  deterministic).
Each case is run at n = max_samples_per_call (the scratch fully used) with a ragged number of MF tiles.
"""
import numpy as np
import pytest
import torch

from gpu_case import F, HALO, make_case, receiver_for

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_06311_b200 as P  # noqa: E402

PAD = 1 << 14   # elements of poison / sentinel on each side


def _run(case, rx, dtype, pad):
    """One device call over the case's core; inputs/outputs embedded in pads when pad > 0."""
    first, n = case["first"], case["n"]
    codes = case["codes"]
    if dtype == "float":
        codes, poison = codes.to(torch.float32), float("nan")
    elif dtype == "uint8":
        poison = 255
    else:
        poison = 32767
    buf = torch.full((codes.numel() + 2 * pad,), poison, dtype=codes.dtype)
    buf[pad:pad + codes.numel()] = codes
    ref = torch.full((n // 4 + 2 * pad,), 0xFF, dtype=torch.uint8)
    ref[pad:pad + n // 4] = case["ref"]
    dec = torch.full((n // 4 + 2 * pad,), 0x5A, dtype=torch.uint8, device="cuda")
    fe = torch.full((2 * n // F + 2 * pad,), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    buf, ref = buf.cuda(), ref.cuda()
    rx.process(buf, first, n, ref=ref[pad:pad + n // 4], decisions=dec[pad:pad + n // 4], offset=pad,
               frame_errors=fe[pad:pad + 2 * n // F])
    z = rx.intermediate(P.KK_STAGE_EQ)[1].cpu()
    y = rx.intermediate(P.KK_STAGE_MF)[1].cpu()
    torch.cuda.synchronize()
    if pad:
        for t, v in ((dec, 0x5A), (fe, 0x5A5A5A5A)):
            assert bool((t[:pad] == v).all()) and bool((t[-pad:] == v).all()), "caller buffer pad overwritten"
    return dict(dec=dec[pad:pad + n // 4].cpu(), fe=fe[pad:pad + 2 * n // F].cpu(), z=z, y=y, stats=rx.stats())


CASES = [
    # name, case kwargs, receiver kwargs, input dtype
    ("blockls_b2b", dict(M=16, dl=0.0, esn0=18.0), {}, "int16"),
    ("blockls_K7", dict(M=4, dl=200000.0, esn0=12.0), {}, "int16"),
    ("blockls_mixed_uint8", dict(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, esn0=26.0),
     dict(input_uint8=True), "uint8"),
    ("blockls_float_lsb", dict(M=64, dl=8000.0, esn0=28.0, sideband=-1), dict(input_float=True), "float"),
    ("ddlms", dict(M=16, dl=112000.0, esn0=18.0, eq_mode="ddlms"), {}, "int16"),
    ("upsample2", dict(M=16, dl=32000.0, esn0=20.0, cspr=8.0, upsample=2), {}, "int16"),
    ("upsample2_uint8_lsb", dict(M=64, dl=8000.0, esn0=26.0, sideband=-1, upsample=2), dict(input_uint8=True),
     "uint8"),
    ("ddlms_max_warmup", dict(M=16, dl=50000.0, esn0=18.0, eq_mode="ddlms", ddlms_block=256, ddlms_warmup=3136),
     {}, "int16"),
    ("mf8192_blockls", dict(M=64, dl=200000.0, esn0=24.0), dict(mf_fft_n=8192), "int16"),
    ("mf8192_ddlms_max_warmup", dict(M=16, dl=50000.0, esn0=18.0, eq_mode="ddlms", ddlms_warmup=2112),
     dict(mf_fft_n=8192), "int16"),
    ("ddlms_warm0_blk4096", dict(M=4, dl=20000.0, esn0=12.0, eq_mode="ddlms", ddlms_block=4096, ddlms_warmup=0),
     {}, "int16"),
    ("static_cd_L5", dict(M=32, dl=200000.0, esn0=20.0, static_cd=True), {}, "int16"),
    ("blockls_K5_prbs", dict(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=112000.0, esn0=22.0,
                             label_source="prbs31"), {}, "int16"),
]


@pytest.mark.parametrize("name,ckw,rkw,dtype", CASES, ids=[c[0] for c in CASES])
def test_guarded_run_is_bit_identical_and_in_bounds(name, ckw, rkw, dtype):
    n = 3 * F
    case = make_case(n=n, first=2 * F, seed=900, **ckw)
    if dtype == "uint8":   # the case generator makes int16 codes; requantise to 8 bits for the uint8 path
        case["codes"] = (case["codes"].to(torch.int32) >> 7).clamp(0, 255).to(torch.uint8)
        case["ocfg"].adc_scale *= 128.0
    rx0 = receiver_for(case, keep=True, max_samples=n, **rkw)
    rx1 = receiver_for(case, keep=True, max_samples=n, debug_guard=True, **rkw)
    a = _run(case, rx0, dtype, pad=0)
    b = _run(case, rx1, dtype, pad=PAD)
    assert rx0.check_guards() == 0                 # guards off: nothing to check
    assert rx1.check_guards() >= 6                 # E, part, clamp, y, z, counters
    assert torch.equal(a["dec"], b["dec"])
    assert torch.equal(a["fe"], b["fe"])
    assert torch.equal(a["z"], b["z"]) and torch.equal(a["y"], b["y"])
    assert a["stats"] == b["stats"]
    assert bool(torch.isfinite(b["z"]).all())
    rx0.close()
    rx1.close()


def test_guarded_host_path_and_repeated_calls():
    n = 2 * F
    case = make_case(M=8, dl=50000.0, esn0=16.0, n=4 * n, first=0, seed=901)
    rx = receiver_for(case, keep=False, max_samples=n, debug_guard=True)
    codes = case["codes"].pin_memory()
    ref = case["ref"].pin_memory()
    dec = torch.zeros(case["n"] // 4, dtype=torch.uint8).pin_memory()
    for c0 in range(0, case["n"], n):
        rx.process_host(codes, c0, n, ref=ref[c0 // 4:(c0 + n) // 4], decisions=dec[c0 // 4:(c0 + n) // 4],
                        offset=c0)
    n_checked = rx.check_guards()
    assert n_checked >= 5 + 6                      # scratch + the two-slot host staging buffers
    st = rx.stats()
    assert st["frames"] == case["n"] // F and st["bad_frames"] == 0
    assert int(np.sum(dec.numpy() != case["ref"].numpy())) == sum(st["sym_err"])   # every decision written
    rx.close()


@pytest.mark.parametrize("eq_mode", ["block_ls", "ddlms"])
def test_guarded_generated_reference(eq_mode):
    """kk_config.ref_prbs: the generated label buffer is canary-guarded too, and counting against it equals
    counting against the caller's label buffer (no ref argument: the generator's labels are used)."""
    n = 3 * F
    case = make_case(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, esn0=16.0, n=n, first=5 * F,
                     seed=902, eq_mode=eq_mode)
    rx0 = receiver_for(case, keep=False, max_samples=n)
    rx1 = receiver_for(case, keep=False, max_samples=n, debug_guard=True, ref_prbs_seed=case["lc"].seed)
    codes = case["codes"].cuda()
    d0 = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
    d1 = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
    rx0.process(codes, case["first"], n, ref=case["ref"].cuda(), decisions=d0)
    rx1.process(codes, case["first"], n, decisions=d1)
    assert rx1.check_guards() >= 6                 # E, part, clamp, y, counters + the generated-label buffer
    assert torch.equal(d0, d1) and rx0.stats() == rx1.stats()
    rx0.close()
    rx1.close()
