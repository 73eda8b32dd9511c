"""CPU: the C-ABI library builds, loads and exports every symbol include/*.h
declares (no compute calls — there is no GPU here)."""
import ctypes as C
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for d, _, files in os.walk(inc):
        for f in files:
            if f.endswith(".h"):
                txt = open(os.path.join(d, f)).read()
                txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
                syms |= set(re.findall(r"\b(smo_[a-z0-9_]+)\s*\(", txt))
    return syms


def test_library_exports_every_declared_symbol():
    from paper_2508_21706_b200 import _lib, build
    build.build()
    lib = C.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing
    # every declared function also has a ctypes signature in the front end
    assert syms <= set(_lib._SIGS), sorted(syms - set(_lib._SIGS))


def test_version_and_error_plumbing_without_gpu():
    from paper_2508_21706_b200 import _lib
    lib = _lib.load()
    assert b"sm_100a" in lib.smo_version()
    # an argument error is reported before any CUDA call
    st = lib.smo_router_topk(None, None, 4, 100, 8, 2, None, None, None, None)
    assert st == _lib.SMO_INVALID_ARG
    assert b"router" in lib.smo_last_error()


def test_sm100a_cubin_contains_tcgen05_and_tma():
    """The shipped kernels are tcgen05/TMA code (SASS UTCHMMA / UTMALDG)."""
    import shutil
    import subprocess
    from paper_2508_21706_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path
