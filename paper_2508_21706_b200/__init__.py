"""B200-native SpecMoEOff speculative verification step (arXiv 2508.21706).

The product is libspecmoe.so (C-ABI: include/specmoe/c_api.h) — hand-written
sm_100a kernels (tcgen05/TMEM/TMA) plus the C++ VerifyEngine and expert
streamer. This package is the thin Python front end:
  * `ops`        torch-tensor wrappers of the kernels (K1-K6),
  * `attention`  mirror of the reference's attention.hpp API,
  * `engine`     VerifyEngine handle (the measured verify step),
  * `build`      the nvcc recipe that produces libspecmoe.so in-tree.
"""
from . import _lib  # noqa: F401

__all__ = ["_lib"]
