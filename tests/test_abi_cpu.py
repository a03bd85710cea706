"""The drop-in boundary: libmlt.so loads, exports every entry point that
include/mlt.h declares (no compute calls without a GPU), and fails loudly —
with a status, not a crash or a silent fallback — when asked for device work
on a machine without a device."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2411_11217_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "mlt.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mlt_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared()
    assert len(names) > 40
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mlt_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = C.CDLL(capi.LIB_PATH)
    for n in names:
        assert getattr(lib, n) is not None


def test_version_and_error_channel(api):
    lib = api.lib
    lib.mlt_version.restype = C.c_char_p
    assert b"sm_100a" in lib.mlt_version()
    with pytest.raises(capi.InfeasiblePolicyError):
        hw = capi.HardwareSpec(1.0, 1e6, 50, 10, 2, 100, 10)
        api.layer_latency(hw, capi.ModelSpec(2, 8, 16, 4, 2, 4, 2, 2.0, 2.0),
                          capi.WorkloadSpec(10, 4), capi.Policy(8, 4, 1, 1, 1.0, 1.0), 10.0)
    assert "exceeds device memory" in api.error()


def test_validate_reports_issues(api):
    lib = api.lib
    f = lib.mlt_validate
    f.restype = C.c_int
    f.argtypes = [C.c_void_p] * 4 + [C.c_char_p, C.c_size_t]
    buf = C.create_string_buffer(512)
    bad = capi.Policy(10, 4, 0, 1, 1.5, 0.3)
    n = f(None, None, None, C.byref(bad), buf, 512)
    assert n == 3  # N % mu, r_w range, r_c without A_g
    assert b"DivisibilityViolation" in buf.value and b"PolicyInconsistency" in buf.value


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="device present")
def test_runtime_without_gpu_fails_loudly():
    from paper_2411_11217_b200.runtime import Runtime
    with pytest.raises(capi.MltError) as e:
        Runtime(capi.ModelSpec(2, 1024, 3584, 8, 2, 8, 2, 2.0, 2.0), capi.Policy(8, 4, 0, 1, 0.0, 0.0),
                budget_bytes=1e9, max_ctx=64)
    assert e.value.code == -6  # MLT_ERR_CUDA: no CPU fallback exists
