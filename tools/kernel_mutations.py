#!/usr/bin/env python
"""Mutation check of the GPU parity suite (diagnostic): each mutation is a plausible mistake in a CUDA kernel
(a wrong sign, a dropped step, a miscount). `--build` (CPU, nvcc cross-compiles) applies each one to a scratch copy
of csrc/ and builds its own library under build/mut/<name>/; `--run` (on the B200) runs a fast subset of the GPU
parity tests against each library (KK_LIB) and reports the mutation "killed" when at least one test fails.
A surviving mutation would mean a kernel step the GPU tests do not pin.

    python tools/kernel_mutations.py --build            # here
    python tools/kernel_mutations.py --run --out profiles/r02_kernel_mutations.json   # on the GPU box
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2104_06311_b200", "csrc")
MUT = os.path.join(ROOT, "build", "mut")

# (name, file, original, mutated, what it breaks)
MUTATIONS = [
    ("k1_hilbert_sign", "k1_kk.cu",
     "v[r] = (r < 16) ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);",
     "v[r] = (r < 16) ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);",
     "K1: Hilbert multiplier +i·sgn instead of −i·sgn"),
    ("k1_magnitude_full_log", "k1_kk.cu",
     "const float m0 = ex2_approx(fmaf(ab0[pos], 0.5f, l2m)), m1 = ex2_approx(fmaf(ab1[pos], 0.5f, l2m));",
     "const float m0 = ex2_approx(fmaf(ab0[pos], 1.0f, l2m)), m1 = ex2_approx(fmaf(ab1[pos], 1.0f, l2m));",
     "K1: |E| = I instead of √I"),
    ("k2_no_carrier_removal", "k2_mf.cu",
     "v[it][r] = cmul(csub(v[it][r], A0), r == 0 ? c : cmul(c, p.rho[r]));",
     "v[it][r] = cmul(v[it][r], r == 0 ? c : cmul(c, p.rho[r]));",
     "K2: carrier estimate A_f not subtracted (tiles inside one frame)"),
    ("k2_fold_drops_alias", "k2_mf.cu",
     "float2 yv = cscale(b, hb);                         // packed: b·hb, then + a·ha (same roundings)",
     "float2 yv = make_float2(0.f, 0.f);",
     "K2: the spectral fold drops the upper half (no aliasing term)"),
    ("k3a_no_agc", "k3_eq.cu",
     "const float g_agc = p0ok ? (float)rsqrt(P0) : 1.0f;", "const float g_agc = 1.0f;",
     "K3a: AGC dropped"),
    ("k3s_ridge_sign", "k3_eq.cu",
     "const double lam = trG * (wl ? (double)p.ridge / (double)N : (double)p.ridge * 0.5 / (double)L);",
     "const double lam = -trG * (wl ? (double)p.ridge / (double)N : (double)p.ridge * 0.5 / (double)L);",
     "K3s: ridge of the wrong sign"),
    ("k3c_no_unbias", "k3_eq.cu",
     "if (isc > 0.0 && isfinite(isc)) sc = (float)isc; else bad = 1;", "if (isc > 0.0 && isfinite(isc)) sc = 1.0f; else bad = 1;",
     "K3c: gain unbias dropped"),
    ("k3c_cpr_sign", "k3_eq.cu",
     "return (rs > 0.f) ? make_float2(cr * rsc, -ci * rsc) : make_float2(sc, 0.f);",
     "return (rs > 0.f) ? make_float2(cr * rsc, ci * rsc) : make_float2(sc, 0.f);",
     "K3c: CPR rotates the wrong way"),
    ("k3c_bits_as_symbols", "k3_eq.cu",
     "          berr += __popc(x);\n", "          berr += __popc(__vcmpne4(x, 0u)) >> 3;\n",
     "K3c: bit errors counted as symbol errors"),
    ("k2_fold_drops_direct", "k2_mf.cu",
     "            ffma2s(yv, ha, a);\n", "",
     "K2: the spectral fold drops the lower half (only the alias)"),
    ("k3a_lag_index", "k3_eq.cu",
     "ffma2s(acc[8 * gg + 4], acc[8 * gg + 5], w[1].x, w[1 + d]);",
     "ffma2s(acc[8 * gg + 4], acc[8 * gg + 5], w[1].x, w[d]);",
     "K3a: odd-base lag sums taken one lag short"),
    ("k3c_cpr_window_local", "k3_eq.cu",
     "        if (p.cpr_window > 512) {                                      // kernel-uniform: windows of W/512 warps",
     "        if (p.cpr_window > 1 << 30) {                                  // kernel-uniform: windows of W/512 warps",
     "K3c: CPR windows above 512 symbols not summed over their warps"),
    ("k3d_update_sign", "k3_ddlms.cu",
     "const float2 m2 = cscale(e, 2.f * mu);             // c += 2μe ⊗ (xr, xi)",
     "const float2 m2 = cscale(e, -2.f * mu);            // c += 2μe ⊗ (xr, xi)",
     "K3′: DDLMS gradient step of the wrong sign"),
    ("kref_prbs_tap", "kref.cu",
     "  const uint32_t n1 = ((w >> 3) ^ w) & m28;                      // b[31 .. 58]",
     "  const uint32_t n1 = ((w >> 2) ^ w) & m28;                      // b[31 .. 58]",
     "kref: PRBS-31 feedback tap x^29 instead of x^28"),
    ("k1u_hilbert_sign", "k1u_kk.cu",
     "v[k] = h ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);",
     "v[k] = h ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);",
     "K1U: Hilbert multiplier +i·sgn instead of −i·sgn (2× upsampling path)"),
    ("k2_ch_fold_alias_dropped", "k2_mf.cu",
     "            cmac2(yv, b, __ldg(&Hc[j + 256 * (r + R3 / 2)]));\n", "",
     "K2 (complex H, static-CD/DDLMS arrangements): the fold's alias term dropped"),
    ("k3a_second_lag_pass_offset", "k3_eq.cu",
     "              lag_acc(acc2, w, LA1, LA - LA1);", "              lag_acc(acc2, w, LA1 - 1, LA - LA1);",
     "K3a (L ≥ 11): the second lag pass starts one lag early"),
    # (Not listed: K3a's silent flag dropped is equivalent on every fp32-reachable input — a frame with
    # P0 ≤ 1e-20·I_ref has y ≡ 0 in fp32, and the unflagged frame's failed solve (θ₀ fallback, counted bad)
    # outputs the same z = 0 and D(0).)
]

TESTS = ["tests/test_gpu_parity.py", "-x", "-q", "-k",
         "c1_b2b or format_parity or q_parity_large or uint8 or linear_only or per_frame_errors or decision_paths "
         "or ddlms_mode_parity or unaligned_reference_labels"]
# the reference-label generator, the upsampling path and the silent-frame rule have their own test files
TESTS_REF = ["tests/test_gpu_refprbs.py", "-x", "-q"]
TESTS_UP = ["tests/test_gpu_upsample.py", "-x", "-q"]


def build(names):
    os.makedirs(MUT, exist_ok=True)
    for name, fn, orig, mut, what in MUTATIONS:
        if names and name not in names:
            continue
        d = os.path.join(MUT, name)
        src = os.path.join(d, "pkg", "csrc")                # kk_host.cpp includes ../../include/kkrx.h
        shutil.rmtree(d, ignore_errors=True)
        shutil.copytree(CSRC, src)
        shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
        p = os.path.join(src, fn)
        text = open(p).read()
        if text.count(orig) != 1:
            print(f"{name:26s} NOT APPLICABLE (pattern count {text.count(orig)})")
            continue
        open(p, "w").write(text.replace(orig, mut))
        env = dict(os.environ, KK_CSRC=src, KK_LIB=os.path.join(d, "libkkrx.so"), KK_BUILD_DIR=os.path.join(d, "obj"))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "paper_2104_06311_b200", "build.py")], env=env,
                           capture_output=True, text=True)
        print(f"{name:26s} {'built' if r.returncode == 0 else 'BUILD FAILED'}")
        if r.returncode != 0:
            print(r.stdout[-1500:] + r.stderr[-1500:])
        shutil.rmtree(os.path.join(d, "obj"), ignore_errors=True)
        shutil.rmtree(os.path.join(d, "pkg"), ignore_errors=True)
        shutil.rmtree(os.path.join(d, "include"), ignore_errors=True)


def run(names, out):
    results = []
    t0 = time.time()                                      # the unmutated library must pass the same subset
    for tests in (TESTS, TESTS_REF, TESTS_UP):
        r = subprocess.run([sys.executable, "-m", "pytest", *tests], cwd=ROOT, capture_output=True, text=True)
        print(f"{'(unmutated library)':26s} {'passes' if r.returncode == 0 else 'FAILS'} {tests[0]} "
              f"({time.time() - t0:.0f} s)", flush=True)
        if r.returncode != 0:
            print(r.stdout[-2000:])
            sys.exit(1)
    for name, fn, orig, mut, what in MUTATIONS:
        if names and name not in names:
            continue
        lib = os.path.join(MUT, name, "libkkrx.so")
        if not os.path.exists(lib):
            results.append(dict(name=name, what=what, status="not-built"))
            continue
        t0 = time.time()
        tests = TESTS_REF if fn == "kref.cu" else TESTS_UP if fn == "k1u_kk.cu" else TESTS
        r = subprocess.run([sys.executable, "-m", "pytest", *tests], cwd=ROOT, env=dict(os.environ, KK_LIB=lib),
                           capture_output=True, text=True)
        failed = [ln.split("::")[1].split()[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
        status = "killed" if r.returncode != 0 else "SURVIVED"
        print(f"{name:26s} {status:8s} {failed[:1]} ({time.time() - t0:.0f} s)", flush=True)
        results.append(dict(name=name, what=what, status=status, first_failing_test=failed[:1],
                            seconds=round(time.time() - t0, 1)))
    if out:
        with open(out, "w") as f:
            json.dump(results, f, indent=1)
    print(json.dumps(results))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--run", action="store_true")
    ap.add_argument("--out", default="")
    ap.add_argument("names", nargs="*")
    a = ap.parse_args()
    if a.build:
        build(a.names)
    if a.run:
        run(a.names, a.out)
