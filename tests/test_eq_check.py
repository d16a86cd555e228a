"""CPU tests of the GPU parity helper `gpu_case.eq_check` (test infrastructure): a frame may miss the 1e-4 EQ
bound only when the oracle, re-run with decisions moved across a slicer boundary they sit on, reproduces it;
any other deviation fails. The "GPU" outputs here are oracle re-runs, so no device is needed."""
import numpy as np
import pytest

from gpu_case import _Decide, _ddlms_block_rerun, _frame_rerun, _near_boundary, eq_check, make_case, run_oracle


def _closest_candidate(calls, M):
    best = None
    for c, zc in enumerate(calls):
        for k, p, t in _near_boundary(zc, M, 1e-2):
            if best is None or t < best[3]:
                best = (c, k, p, t)
    return best


def test_near_boundary_geometry():
    # 16-QAM: levels ±1, ±3 (/√10); a point at I = 2/√10 + 1e-6 sits 1e-6 from the I boundary
    s = 1 / np.sqrt(10)
    z = np.array([(2 + 1e-5) * s + 1j * s, 1 * s + 1j * s])
    c = _near_boundary(z, 16, 1e-5)
    assert len(c) == 1 and c[0][0] == 0 and abs(c[0][1] - (1 * s + 1j * s)) < 1e-12 and abs(c[0][2] - 1e-5 * s) < 1e-12


def test_eq_check_proves_a_training_flip_and_rejects_other_errors():
    case = make_case(M=16, dl=112000.0, cspr=8.0, esn0=14.0, n=4 * 16384, seed=77)
    orc = run_oracle(case)
    cfg = case["ocfg"]
    fi = 2
    _, dec, M = _frame_rerun(orc, cfg, fi, ())
    c, k, p, t = _closest_candidate(dec.calls[:1], M)              # a pass-1 (training) decision
    z_flip, _, _ = _frame_rerun(orc, cfg, fi, ((c, k, p),))
    zg = orc["z"].copy()
    zg[fi * 4096:(fi + 1) * 4096] = z_flip
    raw = np.linalg.norm(z_flip - orc["z"][fi * 4096:(fi + 1) * 4096]) / np.linalg.norm(z_flip)
    assert raw > 1e-5                                               # the flip is visible in the output
    tol = min(1e-4, raw / 2)
    ce, proven, worst = eq_check(zg, orc, cfg, tol=tol, delta=1.01 * t)
    assert [f for f, _ in proven] == [fi] and proven[0][1][0][:2] == (c, k)
    # a deviation that no boundary decision explains is not excused
    zbad = zg.copy()
    zbad[4096:8192] *= 1 + 3 * tol
    with pytest.raises(AssertionError):
        eq_check(zbad, orc, cfg, tol=tol, delta=1.01 * t)
    # nor is the flipped frame when the decision is not within delta of its boundary
    with pytest.raises(AssertionError):
        eq_check(zg, orc, cfg, tol=tol, delta=0.5 * t)


def test_eq_check_ddlms_block_flip():
    case = make_case(M=16, dl=112000.0, cspr=10.0, esn0=15.0, n=2 * 16384, seed=78, eq_mode="ddlms")
    orc = run_oracle(case)
    cfg = case["ocfg"]
    fi, bb = 1, 512
    _, dec, Ms = _ddlms_block_rerun(orc, cfg, fi, bb, ())
    c, k, p, t = _closest_candidate(dec.calls, 16)
    zb, _, _ = _ddlms_block_rerun(orc, cfg, fi, bb, ((c, k, p),))
    zg = orc["z"].copy()
    s0 = fi * 4096 + bb
    zg[s0:s0 + cfg.ddlms_block] = zb
    f0 = fi * 4096
    raw = np.linalg.norm(zg[f0:f0 + 4096] - orc["z"][f0:f0 + 4096]) / np.linalg.norm(orc["z"][f0:f0 + 4096])
    if raw < 1e-7:
        pytest.skip("closest boundary decision does not move this block's outputs")
    tol = min(1e-4, raw / 2)
    _, proven, _ = eq_check(zg, orc, cfg, tol=tol, delta=1.01 * t)
    assert proven and proven[0][:2] == (fi, bb)


def test_decide_hook_default_is_nearest():
    from oracle import constellation as C
    z = np.array([0.3 + 0.1j, -0.9 - 0.2j])
    d = _Decide()
    assert np.array_equal(d(z, 16)[1], C.nearest(z, 16)[1]) and len(d.calls) == 1
