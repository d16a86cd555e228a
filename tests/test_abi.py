"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/kkrx.h declares, its
struct layouts match the binding, and host-only entry points behave (no GPU compute here)."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ensure_built():
    import importlib.util
    spec = importlib.util.spec_from_file_location("kkbuild", os.path.join(ROOT, "paper_2104_06311_b200", "build.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.build()


LIB = _ensure_built()
import paper_2104_06311_b200 as P  # noqa: E402
from oracle import theory  # noqa: E402


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "kkrx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kk_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(LIB)
    names = _declared_functions()
    assert len(names) >= 17
    for n in names:
        assert hasattr(lib, n), n


def test_binding_names_match_header():
    for n in _declared_functions():
        if n in ("kk_config_sizeof", "kk_stats_sizeof"):
            continue
        assert hasattr(P.kkrx, n), n


def test_struct_layouts():
    assert P.kkrx.lib.kk_config_sizeof() == ctypes.sizeof(P.kk_config)
    assert P.kkrx.lib.kk_stats_sizeof() == ctypes.sizeof(P.kk_stats_t) == 8 * P.KK_STATS_WORDS


def test_config_defaults_are_the_papers():
    c = P.kk_config_default()
    assert c.fs_hz == 4e9 and c.baud_hz == 1e9
    assert c.lo_num / c.lo_den * c.fs_hz == pytest.approx(0.516e9)    # PAPER.md:50 tone
    assert c.rolloff == pytest.approx(0.01) and c.rrc_span_sym == 256
    assert (c.hilbert_n, c.hilbert_hop) == (1024, 512)
    assert (c.mf_fft_n, c.mf_hop, c.frame_symbols) == (4096, 3072, 4096)
    assert c.eq_widely_linear == 1 and c.cpr_window == 256


def test_q_from_ber_matches_oracle_theory():
    for ber in (0.3, 3e-2, 1e-3, 2.27e-4, 1e-7):
        assert P.kk_q_from_ber(ber) == pytest.approx(theory.q_from_ber(ber), abs=1e-9)
    for bad in (0.0, 0.5, 1.0, -1.0):
        with pytest.raises(P.KKError) as e:
            P.kk_q_from_ber(bad)
        assert e.value.status == P.KK_ERR_DOMAIN


@pytest.mark.parametrize("field,value", [("cpr_window", 100), ("hilbert_n", 2048), ("fs_hz", 8e9),
                                         ("eq_taps", 4), ("eq_taps", 99), ("default_format", 128),
                                         ("max_samples_per_call", 1000), ("sideband", 0), ("lo_den", 0),
                                         ("rrc_span_sym", 512), ("ref_intensity", 0.0),
                                         ("debug_guard", 2)])
def test_invalid_configs_rejected_before_any_cuda_call(field, value):
    c = P.kk_config_default()
    setattr(c, field, value)
    with pytest.raises(P.KKError) as e:
        P.kk_init(c)
    assert e.value.status == P.KK_ERR_CONFIG


@pytest.mark.parametrize("warmup", [3200, 100, -64])
def test_ddlms_warmup_bound(warmup):
    """K2's outermost tiles must stay inside E (core ± one frame): 2·(2W + 2) + 2·1536 − 2 + 512 ≤ 16384
    ⇒ W ≤ 3136 (multiple of 64)."""
    c = P.kk_config_default()
    c.eq_mode = P.KK_EQ_DDLMS
    c.ddlms_warmup = warmup
    with pytest.raises(P.KKError) as e:
        P.kk_init(c)
    assert e.value.status == P.KK_ERR_CONFIG


def test_strerror_and_null_handling():
    for s in range(-8, 1):
        assert isinstance(P.kk_strerror(s), str) and P.kk_strerror(s)
    assert P.kkrx.lib.kk_halo(None, None, None) == P.KK_ERR_NULL
    assert P.kkrx.lib.kk_stats(None, None) == P.KK_ERR_NULL
    assert P.kkrx.lib.kk_process_frames(None, None, 0, 16384, None, None, None) == P.KK_ERR_NULL
    assert P.kkrx.lib.kk_check_guards(None, None) == P.KK_ERR_NULL
    P.kkrx.lib.kk_destroy(None)


def test_stats_word_decoder():
    w = list(range(24))
    d = P.stats_from_words(w)
    assert d["sym"] == [0, 1, 2, 3, 4] and d["bit_err"] == [15, 16, 17, 18, 19] and d["bad_frames"] == 23
