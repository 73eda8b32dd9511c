"""Build recipe for libspecmoe.so (sm_100a) — in-tree, so the .so travels to
the GPU box with the gpurun snapshot. Used by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libspecmoe.so")
SOURCES = ["c_api.cu", "ops.cu", "gemm_tc.cu", "moe_tc.cu", "attention.cu", "engine.cu", "decode.cu", "prefill.cu", "streamer.cu",
           "ep.cu", "xfer.cu", "tcode.cu"]
CXX_SOURCES = ["cpu_attn.cpp"]  # host code (CPU attention placement), g++ with AVX2/FMA
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-O3", "-mavx2", "-mfma", "-std=c++17", "-fPIC", "-pthread", "-I", CSRC]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
         "-I", CSRC]


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, jobs: int = 8) -> str:
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "cpu_attn.h"), os.path.join(CSRC, "engine.cuh"), os.path.join(CSRC, "tcode.cuh"),
               os.path.join(ROOT, "include", "specmoe", "c_api.h")]
    procs, objs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if _stale(o, [s] + headers):
            cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        while len([p for _, p in procs if p.poll() is None]) >= jobs:
            procs[0][1].wait()
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cpp", ".o"))
        objs.append(o)
        if _stale(o, [s] + headers):
            cmd = [CXX, *CXX_FLAGS, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd))
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    errs = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            errs.append(f"{src}:\n{out.decode()}")
        elif verbose and out:
            print(out.decode())
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    if _stale(OUT, objs):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", OUT, *objs,
               "-Xcompiler", "-pthread"]
        subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
