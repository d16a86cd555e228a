import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from gpu_case import make_case, run_gpu, run_oracle
case = make_case(M=16, dl=112000.0, cspr=6.0, esn0=18.0, noise="white", n=1 << 17, seed=112, upsample=2)
g, o = run_gpu(case), run_oracle(case)
z, zo = g["z"].reshape(-1, 4096), o["z"].reshape(-1, 4096)
fe = np.linalg.norm(z - zo, axis=1) / np.linalg.norm(zo, axis=1)
print("per-frame z rel err", np.array2string(fe, precision=2))
print("dec agree", np.mean(g["dec"] == o["dec"]), "ser", np.mean(o["dec"] != case["ref"].numpy()))
