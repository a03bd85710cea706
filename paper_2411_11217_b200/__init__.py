"""B200-native MoE-Lightning decode hot path.

The product is the native library libmlt.so (C ABI: include/mlt.h) built
from csrc/ — C++20 host (lightplan planner/scheduler API, runtime, host
attention) and hand-written sm_100a kernels.  This package only binds it:
`capi` (ctypes mirror of mlt.h) and `runtime` (the decode runtime handle).
Importing fails loudly if the library has not been built.
"""
from . import capi  # noqa: F401

capi.load_product()
