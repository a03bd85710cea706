"""Shared fixtures.  `gpu` marks tests that need a B200 (run by the driver
with -m gpu on a GPU box); everything else runs on CPU."""
import ctypes as C
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2411_11217_b200 import capi  # noqa: E402

REF_SO = os.path.join(ROOT, "oracle", "_ref", "liblightplan_ref.so")
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


@pytest.fixture(scope="session")
def api():
    return capi.load_product()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference lightplan (oracle/_ref) behind the same C structs."""
    if not os.path.exists(REF_SO):
        pytest.fail(f"{REF_SO} missing; build it with `make -C oracle ref` (needs /root/reference)")
    extra = {"oracle_layer_latency": (C.c_int, [C.POINTER(capi.HardwareSpec),
                                                C.POINTER(capi.ModelSpec),
                                                C.POINTER(capi.Policy), C.c_double,
                                                C.POINTER(C.c_double)]),
             "replay_simulate": (C.c_int, [C.c_void_p, C.POINTER(capi.TimelineEntry),
                                           C.POINTER(C.c_double), C.POINTER(C.c_double)]),
             "brute_force_search": (C.c_int, [C.POINTER(capi.HardwareSpec), C.POINTER(capi.ModelSpec),
                                              C.POINTER(capi.WorkloadSpec), C.POINTER(capi.SearchGrid),
                                              C.POINTER(capi.Policy), C.POINTER(C.c_double)]),
             "replay_batching": (C.c_int, [C.POINTER(C.c_char_p), C.POINTER(C.c_int64), C.c_int32,
                                           C.POINTER(capi.BatchParams), C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32)])}
    return capi.Api(C.CDLL(REF_SO), "ref_", extra)


# ---- fixtures mirroring proj/tests/support/fixtures.hpp -------------------
def toy_model():
    return capi.ModelSpec(2, 8, 16, 4, 2, 4, 2, 2.0, 2.0)


def toy_hardware():
    return capi.HardwareSpec(1e6, 1e6, 50.0, 10.0, 2.0, 100.0, 10.0)


def toy_workload():
    return capi.WorkloadSpec(10, 4)


def toy_policy():
    return capi.Policy(8, 4, 0, 1, 0.0, 0.0)


def mixtral_8x22b_model():
    return capi.ModelSpec(56, 6144, 16384, 48, 8, 8, 2, 2.0, 2.0)


def mixtral_8x7b_model():
    return capi.ModelSpec(32, 4096, 14336, 32, 8, 8, 2, 2.0, 2.0)
