#!/usr/bin/env python
"""Mutation check of the oracle's pins (test infrastructure; CPU only).

Each mutation below is a plausible mistake in `oracle/` — a dropped term, a wrong sign or index, a
sub-frame grid, a missing step. For each, a scratch copy of `oracle/`, `kkgen/` and `tests/` is mutated and
`tests/test_oracle_pins.py` is run; the mutation is "killed" if at least one pin fails. A surviving
mutation means a reading the pins do not fix ("parity unpinned").

    python tools/oracle_mutations.py [name ...]      # all by default; prints one line per mutation + JSON
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, file, original text, mutated text, what it breaks)
MUTATIONS = [
    ("r8_per_block_mean", "oracle/receiver.py",
     "    A = E.reshape(-1, F).mean(axis=1)\n    return E - np.repeat(A, F), A",
     "    A = E.reshape(-1, F).mean(axis=1)\n    Ab = E.reshape(-1, 512).mean(axis=1)\n    return E - np.repeat(Ab, 512), A",
     "R8: carrier estimate per 512-sample block instead of per frame"),
    ("r8_no_removal", "oracle/receiver.py",
     "    return E - np.repeat(A, F), A",
     "    return E.copy(), A",
     "R8: no carrier removal"),
    ("r27_no_unbias", "oracle/receiver.py",
     "    u, gam, ok = o8_unbias(y1, M, decide)\n",
     "    u, gam, ok = y1, 1.0, True\n",
     "R27: gain unbias deleted"),
    ("r2_hilbert_sign", "oracle/receiver.py",
     "mult = np.where((q > 0) & (q < N // 2), -1j, np.where(q > N // 2, 1j, 0.0))\n    phi = np.empty",
     "mult = np.where((q > 0) & (q < N // 2), 1j, np.where(q > N // 2, -1j, 0.0))\n    phi = np.empty",
     "R2: Hilbert multiplier sign"),
    ("r1_keep_first_half", "oracle/receiver.py",
     "blk[lead:lead + hop]", "blk[0:hop]",
     "R1: OLS keeps the first hop samples instead of the centre"),
    ("o2_no_half", "oracle/receiver.py",
     "return 0.5 * np.log(Ic), np.sqrt(Ic), clamped", "return np.log(Ic), np.sqrt(Ic), clamped",
     "O2: ln I instead of ½ ln I"),
    ("r9_lo_sign", "oracle/receiver.py",
     "return e * np.exp(-2j * np.pi * cfg.sideband * q / cfg.lo_den)",
     "return e * np.exp(2j * np.pi * cfg.sideband * q / cfg.lo_den)",
     "R9: LO shifts the wrong way"),
    ("r6_odd_decimation", "oracle/receiver.py",
     "n = 2 * np.arange(m0, m1, dtype=np.int64)", "n = 2 * np.arange(m0, m1, dtype=np.int64) + 1",
     "R6: decimation keeps the odd phase"),
    ("r10_ridge_to_zero", "oracle/receiver.py",
     "np.linalg.solve(Lc, p + lam * th0)", "np.linalg.solve(Lc, p)",
     "R10: ridge pulls toward 0 instead of θ₀"),
    ("r10_no_conj_branch", "oracle/receiver.py",
     "Phi = np.concatenate([U, np.conj(U)], axis=1) if wl else U",
     "Phi = np.concatenate([U, U], axis=1) if wl else U",
     "R10: widely-linear branch uses u instead of conj(u)"),
    ("r12_cpr_sign", "oracle/receiver.py",
     "return u * np.repeat(np.exp(-1j * th), W), th", "return u * np.repeat(np.exp(1j * th), W), th",
     "R12: CPR rotates the wrong way"),
    ("r25_no_agc", "oracle/receiver.py",
     "    th0 = g * th0\n", "    th0 = th0\n",
     "R25: AGC dropped"),
    ("o11_q_no_sqrt2", "oracle/theory.py",
     "return 20.0 * math.log10(math.sqrt(2.0) * special.erfcinv(2.0 * ber))",
     "return 20.0 * math.log10(special.erfcinv(2.0 * ber))",
     "O11: Q without the √2"),
    ("r13_gray_16", "oracle/constellation.py",
     "labs.append((_gray(iI) << half_bits) | _gray(iQ))", "labs.append((iI << half_bits) | _gray(iQ))",
     "R13: natural instead of Gray labels on I"),
    # (Not listed: the Hilbert multiplier's Nyquist bin set to ±i instead of 0 is an equivalent mutant — for real
    # input X[N/2] is real, i·X[N/2] contributes a purely imaginary (−1)^n term that `.real` discards.)
    ("r4_rolloff_x10", "oracle/receiver.py",
     "    b = cfg.rolloff\n    h = np.zeros(2 * half + 1)", "    b = 10 * cfg.rolloff\n    h = np.zeros(2 * half + 1)",
     "R4: RRC roll-off 10 % instead of 1 %"),
    ("r4_rrc_denominator", "oracle/receiver.py",
     "h[idx] = num / (math.pi * t * (1 - (4 * b * t) ** 2))", "h[idx] = num / (math.pi * t)",
     "R4: RRC impulse response without its (1 − (4βt)²) denominator"),
    ("r12_cpr_half_window", "oracle/receiver.py",
     "    s = (u * np.conj(d)).reshape(-1, W).sum(axis=1)\n    th = np.where(s != 0, np.angle(s), 0.0)\n    return u * np.repeat(np.exp(-1j * th), W), th",
     "    s = (u * np.conj(d)).reshape(-1, W // 2).sum(axis=1)\n    th = np.where(s != 0, np.angle(s), 0.0)\n    return u * np.repeat(np.exp(-1j * th), W // 2), th",
     "R12: CPR windows of W/2 symbols"),
    ("r9_lo_frequency", "oracle/receiver.py",
     "q = np.mod(cfg.lo_num * np.mod(n, cfg.lo_den), cfg.lo_den)",
     "q = np.mod((cfg.lo_num - 1) * np.mod(n, cfg.lo_den), cfg.lo_den)",
     "R9: LO at 0.512 instead of 0.516 GHz"),
    ("r7_eps_not_scaled", "oracle/receiver.py",
     "def o2_front_end(I: np.ndarray, cfg: OracleConfig):\n    eps = cfg.clamp_rel * cfg.ref_intensity",
     "def o2_front_end(I: np.ndarray, cfg: OracleConfig):\n    eps = cfg.clamp_rel",
     "R7: clamp floor ε without the I_ref scale"),
    ("r25_agc_no_sqrt", "oracle/receiver.py",
     "    g = 1.0 / math.sqrt(P0)\n", "    g = 1.0 / P0\n",
     "R25: AGC gain 1/P0 instead of 1/√P0"),
    ("r10_ridge_unnormalised", "oracle/receiver.py",
     "lam = cfg.eq_ridge * np.real(np.trace(R)) / n_par", "lam = cfg.eq_ridge * np.real(np.trace(R))",
     "R10: ridge λ = ridge·tr(R) without the 1/(2L)"),
    ("r27_unbias_by_output_power", "oracle/receiver.py",
     "gam = np.sum(y1 * np.conj(d1)) / np.sum(np.abs(d1) ** 2)", "gam = np.sum(y1 * np.conj(d1)) / np.sum(np.abs(y1) ** 2)",
     "R27: γ normalised by the output power instead of the decisions'"),
    ("r10_training_on_unscaled", "oracle/receiver.py",
     "    # (4) pass 1 and decisions\n    y0 = Phi @ th0\n", "    # (4) pass 1 and decisions\n    y0 = Phi @ (th0 / g)\n",
     "R10/R25: training decisions on the pass-1 output before the AGC"),
    ("o1_offset_sign", "oracle/receiver.py",
     "return cfg.adc_scale * (codes.astype(np.float64) - cfg.adc_offset)",
     "return cfg.adc_scale * (codes.astype(np.float64) + cfg.adc_offset)",
     "O1: ADC offset added instead of subtracted"),
    ("r9_lo_phase_origin", "oracle/receiver.py",
     "    q = np.mod(cfg.lo_num * np.mod(n, cfg.lo_den), cfg.lo_den)\n    return e",
     "    q = np.mod(cfg.lo_num * np.mod(n + 1, cfg.lo_den), cfg.lo_den)\n    return e",
     "R9: LO phase origin one sample off the global grid"),
    ("r4_half_span", "oracle/receiver.py",
     "    half = cfg.rrc_span_sym * sps // 2\n", "    half = cfg.rrc_span_sym * sps // 4\n",
     "R4: RRC truncated to half the span"),
    ("o10_bits_as_symbols", "oracle/receiver.py",
     "frame_err[fi] = (int(np.sum(lab != r)), int(np.sum(popcount(lab ^ r))))",
     "frame_err[fi] = (int(np.sum(lab != r)), int(np.sum(lab != r)))",
     "O10: bit errors counted as symbol errors"),
    ("r13_qam_norm", "oracle/constellation.py",
     "norm = math.sqrt(2.0 * (M - 1) / 3.0)", "norm = math.sqrt(2.0 * (M - 1) / 3.0) * 1.05",
     "R13: square-QAM points not at unit mean energy"),
    ("next2_cd_sign", "oracle/receiver.py",
     "    nu = np.fft.fftfreq(N, d=1.0 / cfg.fs_hz)\n    f_c = cfg.fs_hz * cfg.lo_num / cfg.lo_den\n    C = np.exp(-1j * (beta2L(cfg) / 2) * (2 * np.pi * (nu + cfg.sideband * f_c)) ** 2)",
     "    nu = np.fft.fftfreq(N, d=1.0 / cfg.fs_hz)\n    f_c = cfg.fs_hz * cfg.lo_num / cfg.lo_den\n    C = np.exp(1j * (beta2L(cfg) / 2) * (2 * np.pi * (nu + cfg.sideband * f_c)) ** 2)",
     "NEXT-2: static filter applies CD instead of its inverse"),
    ("next2_cd_no_carrier_ref", "oracle/receiver.py",
     "    nu = np.fft.fftfreq(N, d=1.0 / cfg.fs_hz)\n    f_c = cfg.fs_hz * cfg.lo_num / cfg.lo_den\n    C = np.exp(-1j * (beta2L(cfg) / 2) * (2 * np.pi * (nu + cfg.sideband * f_c)) ** 2)",
     "    nu = np.fft.fftfreq(N, d=1.0 / cfg.fs_hz)\n    f_c = cfg.fs_hz * cfg.lo_num / cfg.lo_den\n    C = np.exp(-1j * (beta2L(cfg) / 2) * (2 * np.pi * nu) ** 2)",
     "NEXT-2: CD inverse referenced to baseband instead of the carrier"),
    ("r5_theta0_cd_sign", "oracle/receiver.py",
     "    A = np.exp(-2j * np.pi * np.outer(nu, j) / (2 * cfg.baud_hz))\n    C = np.exp(-1j * (beta2L(cfg) / 2) * (2 * np.pi * (nu + cfg.sideband * f_c)) ** 2)",
     "    A = np.exp(-2j * np.pi * np.outer(nu, j) / (2 * cfg.baud_hz))\n    C = np.exp(1j * (beta2L(cfg) / 2) * (2 * np.pi * (nu + cfg.sideband * f_c)) ** 2)",
     "θ₀: the initial FIR approximates CD instead of its inverse"),
    ("seq_ddlms_update_sign", "oracle/receiver.py",
     "        out[i] = o\n        w = w + mu * e * np.conj(x)\n", "        out[i] = o\n        w = w - mu * e * np.conj(x)\n",
     "NEXT-1: sequential DDLMS gradient step of the wrong sign"),
    ("seq_ddlms_v_branch", "oracle/receiver.py",
     "        if cfg.eq_widely_linear:\n            v = v + mu * e * x\n        cnt += 1",
     "        if cfg.eq_widely_linear:\n            v = v + mu * e * np.conj(x)\n        cnt += 1",
     "NEXT-1: widely-linear branch updated with conj(x)"),
    ("r26_schedule_shift", "oracle/receiver.py",
     "return int(self.formats[(f // self.segment_frames) % len(self.formats)])",
     "return int(self.formats[((f + 1) // self.segment_frames) % len(self.formats)])",
     "R26: format schedule one frame early"),
    ("pu_halfband_centre", "oracle/receiver.py",
     "    f[k == 0] = 0.5\n", "    f[k == 0] = 1.0\n",
     "KK upsampling: half-band centre tap 1 instead of ½ (DC gain 1.5)"),
    ("silent_threshold_absolute", "oracle/receiver.py",
     "if not (P0 > cfg.p0_min_rel * cfg.ref_intensity and np.isfinite(P0)):",
     "if not (P0 > cfg.p0_min_rel and np.isfinite(P0)):",
     "silent-frame rule: power threshold not relative to I_ref"),
    # (Not listed: the restart form's μ schedule reversed — μ_warm on the kept symbols — still passes the
    # restart-vs-sequential pin (≥ 99.9 % identical decisions, Q within 0.1 dB): at the pinned shapes the
    # schedule's effect (steady-state misadjustment ∝ μ) is below the pins' resolution. A tuning reading.)
    ("p11_noise_per_axis", "oracle/theory.py",
     "sig = math.sqrt(n0 / 2.0)                         # per-axis std",
     "sig = math.sqrt(n0)                               # per-axis std",
     "P11: closed-form BER with the full N0 on each axis"),
    ("p11_natural_labels", "oracle/theory.py",
     "e_axis = sum(P[i, j] * _hd(gray(i), gray(j)) for i in range(m) for j in range(m)) / m",
     "e_axis = sum(P[i, j] * _hd(i, j) for i in range(m) for j in range(m)) / m",
     "P11: closed-form square-QAM BER with natural instead of Gray label distances"),
    ("p11_8qam_bits", "oracle/theory.py",
     "return (eI + eQ) / 3.0", "return (eI + eQ) / 2.0",
     "P11: 8-QAM BER divided by 2 bits instead of 3"),
    ("seq_ddlms_no_carry", "oracle/receiver.py",
     "            seq_state = seq_next\n", "            seq_state = None\n",
     "NEXT-1: sequential DDLMS state not carried across frames"),
]


def run(names):
    results = []
    for name, rel, old, new, what in MUTATIONS:
        if names and name not in names:
            continue
        tmp = tempfile.mkdtemp(prefix=f"mut_{name}_")
        try:
            for d in ("oracle", "kkgen", "tests"):
                shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                                ignore=shutil.ignore_patterns("__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
            p = os.path.join(tmp, rel)
            src = open(p).read()
            if src.count(old) != 1:
                results.append(dict(name=name, what=what, status="not-applicable"))
                print(f"{name:24s} NOT APPLICABLE (pattern count {src.count(old)})", flush=True)
                continue
            open(p, "w").write(src.replace(old, new))
            t = time.time()
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q",
                                "-p", "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
            failed = [ln.split("::", 1)[1].split(" ")[0] for ln in r.stdout.splitlines()
                      if ln.startswith("FAILED")]
            status = "killed" if r.returncode != 0 else "SURVIVED"
            results.append(dict(name=name, what=what, status=status, first_failing_pin=failed[:1],
                                seconds=round(time.time() - t, 1)))
            print(f"{name:24s} {status:8s} {failed[:1]} ({time.time() - t:.0f} s)", flush=True)
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
    print(json.dumps(results))
    return results


if __name__ == "__main__":
    res = run(sys.argv[1:])
    sys.exit(0 if all(r["status"] != "SURVIVED" for r in res) else 1)
