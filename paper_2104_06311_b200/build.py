"""Build libkkrx.so in-tree with nvcc for sm_100a (no torch involved).

    python paper_2104_06311_b200/build.py        # or __graft_entry__.build() (does not import the package)
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# A/B experiments only (tools/ab_dirs.sh): another source tree, object directory and library path
CSRC = os.environ.get("KK_CSRC", os.path.join(HERE, "csrc"))
LIB = os.environ.get("KK_LIB", os.path.join(HERE, "libkkrx.so"))
BUILD = os.environ.get("KK_BUILD_DIR", os.path.join(ROOT, "build"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
# diagnostics only (e.g. KK_NVCC_DEFINES=-DKK_PHASE_TIMING with --force); never set for a measured build
FLAGS += os.environ.get("KK_NVCC_DEFINES", "").split()
SOURCES = ["k1_kk.cu", "k1u_kk.cu", "k2_mf.cu", "k3_eq.cu", "k3_ddlms.cu", "kref.cu", "kk_host.cpp"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    # the compile flags (incl. KK_NVCC_DEFINES) are part of every object's identity: a change rebuilds all
    stamp = os.path.join(BUILD, "flags.stamp")
    want = " ".join([NVCC] + ARCH + FLAGS)
    if not os.path.exists(stamp) or open(stamp).read() != want:
        force = True
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "kkrx.h"))
    objs = []
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or not _newer(obj, [src] + headers):
            cmd = [NVCC] + ARCH + FLAGS + ["-Xptxas", "-v", "-c", src, "-o", obj]
            jobs.append((s, cmd))

    def run(job):
        name, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(BUILD, name + ".ptxas.log"), "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr[-4000:]}")
        return name

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for name in ex.map(run, jobs):
            if verbose:
                print("compiled", name)
    if force or jobs or not _newer(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    with open(stamp, "w") as f:
        f.write(want)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
