"""Probe: GPU-vs-oracle parity at very low CSPR (minimum-phase condition violated, many near-zero
intensities) — decision agreement, per-frame EQ error, field error."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from gpu_case import field_rel_err, make_case, rel, run_gpu, run_oracle
for M, cspr, esn0, up in ((16, 0.0, 18.0, 1), (16, 2.0, 18.0, 1), (4, 1.0, 12.0, 1), (16, 2.0, 18.0, 2), (64, 4.0, 26.0, 1)):
    case = make_case(M=M, dl=32000.0, cspr=cspr, esn0=esn0, n=1 << 17, seed=141, upsample=up)
    g, o = run_gpu(case), run_oracle(case)
    z, zo = g["z"].reshape(-1, 4096), o["z"].reshape(-1, 4096)
    fe = np.linalg.norm(z - zo, axis=1) / np.linalg.norm(zo, axis=1)
    print(dict(M=M, cspr=cspr, up=up, field=float(field_rel_err(g, o)), mf=float(rel(g["y"], o["y"])),
               agree=float(np.mean(g["dec"] == o["dec"])), ser=float(np.mean(o["dec"] != case["ref"].numpy())),
               clamped=o["counts"]["clamped"], eq_frames=np.array2string(fe, precision=1)), flush=True)
