"""paper_2602_22158_b200 — B200-native checkpoint tailoring (LLMTailor hot path).

The product is ``libtailor_b200.so`` (C ABI: include/tailor_b200.h; C++ engine
+ sm_100a kernels) and the ``bin/tailor`` CLI. This package is the Python
binding used by the tests and ``bench.py``; it loads the in-tree library and
raises if it is missing (there is no Python or CPU fallback).
"""
from ._lib import CLI_PATH, LIB_PATH, ErrorKind, TailorError, lib  # noqa: F401
from .tailor import *  # noqa: F401,F403
