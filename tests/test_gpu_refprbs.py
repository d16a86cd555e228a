"""GPU: the reference labels generated in the receiver (kk_config.ref_prbs, include/kkrx.h) are the transmitter's
sequence bit for bit — the error counters and decisions equal those of the same stream counted against the
label buffer from kkgen, on the device path, the host path and the DDLMS path (PAPER.md:112 BER against the
known transmitted sequence; DESIGN.md §4 for the sequence)."""
import pytest
import torch

from gpu_case import F, make_case, receiver_for

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _run(case, rx, with_ref, host=False):
    first, n = case["first"], case["n"]
    dec = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
    if host:
        codes = case["codes"].pin_memory()
        ref = case["ref"].pin_memory() if with_ref else None
        hdec = torch.zeros(n // 4, dtype=torch.uint8).pin_memory()
        rx.process_host(codes, first, n, ref=ref, decisions=hdec)
        dec = hdec
    else:
        rx.process(case["codes"].cuda(), first, n, ref=case["ref"].cuda() if with_ref else None, decisions=dec)
    return rx.stats(), dec.cpu()


@pytest.mark.parametrize("first,eq_mode,host,kind", [(5 * F, "block_ls", False, "hash"),
                                                     ((1 << 34) + 3 * F, "block_ls", False, "hash"),
                                                     (5 * F, "block_ls", True, "hash"), (7 * F, "ddlms", False, "hash"),
                                                     (5 * F, "block_ls", False, "prbs31"),
                                                     ((1 << 36) + 9 * F, "block_ls", True, "prbs31"),
                                                     (7 * F, "ddlms", False, "prbs31")])
def test_generated_reference_equals_label_buffer(first, eq_mode, host, kind):
    """Mixed 4/8/16/32/64-QAM (one format per frame) with errors; symbol indices past 2^32 exercise the hash's
    high word and, for the ITU-T PRBS-31 stream (kk_config.ref_prbs = 2), the jump-ahead past many periods."""
    case = make_case(formats=(4, 8, 16, 32, 64), segment_frames=1, dl=32000.0, cspr=10.0, esn0=14.0, n=10 * F,
                     first=first, seed=977, eq_mode=eq_mode, label_source=kind)
    s_buf, d_buf = _run(case, receiver_for(case, keep=False), True, host)
    rx = receiver_for(case, keep=False, ref_prbs_seed=case["lc"].seed, ref_prbs_kind=kind)
    s_gen, d_gen = _run(case, rx, False, host)
    assert sum(s_buf["sym_err"]) > 0 and sum(s_buf["sym"]) == 10 * F // 4
    for k in ("sym", "sym_err", "bits", "bit_err"):
        assert list(s_gen[k]) == list(s_buf[k]), k
    assert torch.equal(d_gen, d_buf)
    # a label buffer still wins over the generator
    s_both, _ = _run(case, receiver_for(case, keep=False, ref_prbs_seed=case["lc"].seed ^ 1, ref_prbs_kind=kind), True,
                     host)
    assert list(s_both["sym_err"]) == list(s_buf["sym_err"])
