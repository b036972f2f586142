"""Build libpoly_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python paper_1609_01882_b200/build.py

Objects and the ptxas resource report go to paper_1609_01882_b200/build/;
the shared library lands next to this file so it travels with the repo
snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libpoly_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["capi.cu", "capi_ivf.cu", "kernels_encode.cu", "kernels_scan.cu", "kernels_topk.cu", "kernels_ivf.cu",
           "kernels_rescue.cu", "kernels_coarse.cu", "kernels_ivf_scan.cu", "capi_multi.cu", "capi_kmeans.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", f"-I{os.path.join(os.path.dirname(HERE), 'include')}"]


def _stale(obj, deps):
    return not os.path.exists(obj) or any(os.path.getmtime(d) > os.path.getmtime(obj) for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "poly_b200.h"))
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        objs.append(o)
        if _stale(o, [s] + headers):
            r = subprocess.run([NVCC, *FLAGS, "-c", s, "-o", o], capture_output=True, text=True)
            with open(os.path.join(OUT_DIR, src.replace(".cu", ".ptxas.log")), "w") as f:
                f.write(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
    if _stale(LIB, objs):
        subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", LIB,
                        "-lcudart"], check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
