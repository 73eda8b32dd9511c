"""Compile the reference's OWN unit suites and acceptance gate (sources read
in place from /root/reference/proj/tests, never copied) against this repo's
drop-in headers (include/moeplan) + the doctest shim (tests/cpp/doctest.h).

Outputs go to build/refsuites/ (git-ignored; travels to the GPU box with the
gpurun snapshot). test_attention and acceptance call moeplan::chunked_attention,
which runs on the GPU through libspecmoe.so, so they are run by the gpu tier.
Also builds `control_*` binaries against the reference headers themselves, so
assertion counts can be compared one-for-one.
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_TESTS = "/root/reference/proj/tests"
REF_INC = "/root/reference/proj/include"
JSON = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
OUT = os.path.join(ROOT, "build", "refsuites")
CPU_SUITES = ["test_config", "test_roofline", "test_memory", "test_pipeline", "test_specdec", "test_optimizer"]
GPU_SUITES = ["test_attention", "acceptance"]


def available() -> bool:
    return os.path.isdir(REF_TESTS) and os.path.isdir(JSON)


def _compile(src, out, inc, link_lib):
    cmd = ["g++", "-std=c++20", "-O2", f"-I{inc}", f"-I{os.path.join(ROOT, 'tests', 'cpp')}",
           f"-I{os.path.join(ROOT, 'include')}", f"-I{JSON}", src, "-o", out]
    if link_lib:
        libdir = os.path.join(ROOT, "paper_2508_21706_b200")
        cmd += [f"-L{libdir}", "-lspecmoe", "-Wl,-rpath,$ORIGIN/../../paper_2508_21706_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile {src} failed:\n{r.stderr[-4000:]}")


def build(control: bool = True) -> list[str]:
    if not available():
        return []
    os.makedirs(OUT, exist_ok=True)
    built = []
    ours = os.path.join(ROOT, "include")
    for name in CPU_SUITES + GPU_SUITES:
        src = os.path.join(REF_TESTS, name + ".cpp")
        gpu = name in GPU_SUITES
        out = os.path.join(OUT, name)
        if not os.path.exists(out) or os.path.getmtime(out) < max(
                os.path.getmtime(src), *[os.path.getmtime(os.path.join(ours, "moeplan", f))
                                         for f in os.listdir(os.path.join(ours, "moeplan"))]):
            _compile(src, out, ours, link_lib=gpu)
        built.append(out)
        if control and not gpu:
            cout = os.path.join(OUT, "control_" + name)
            if not os.path.exists(cout):
                _compile(src, cout, REF_INC, link_lib=False)
    return built


if __name__ == "__main__":
    print("\n".join(build()) or "reference tests not available", file=sys.stderr)


OWN_GPU_SUITES = ["test_verify_engine"]
OWN_CPU_SUITES = ["test_profile_csv", "test_plan_memory"]


def build_own() -> list[str]:
    """This repository's own C++ suites (need only the image's toolchain)."""
    os.makedirs(OUT, exist_ok=True)
    built = []
    for name in OWN_GPU_SUITES + OWN_CPU_SUITES:
        src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
        out = os.path.join(OUT, name)
        inc = os.path.join(ROOT, "include")
        deps = [src, os.path.join(inc, "specmoe", "c_api.h")] + [
            os.path.join(inc, "moeplan", f) for f in os.listdir(os.path.join(inc, "moeplan"))]
        if not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(d) for d in deps):
            if not os.path.isdir(JSON):
                continue
            _compile(src, out, inc, link_lib=name in OWN_GPU_SUITES)
        built.append(out)
    return built
