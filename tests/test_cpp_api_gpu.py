"""The reference-style C++ API additions (include/lightplan/runtime.hpp;
SURVEY.md §8(b)): a plain C++20 program (tests/cpp/execute_demo.cpp) built
against include/lightplan/*.hpp and libmlt.so builds the schedule with the
reference's build_schedule, runs it with sim::execute, checks the measured
timeline with metrics()/verify_timeline(), calls decode_layer, and hits the
error conventions.  Its greedy ids must equal the same decode through the C
ABI (Runtime.decode) bit for bit, and mlt_runtime_execute (the C form of
sim::execute) must agree too."""
import json
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_11217_b200 import capi  # noqa: E402
from paper_2411_11217_b200.runtime import Runtime  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2411_11217_b200")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cpp") / "execute_demo")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "execute_demo.cpp"), "-L", PKG, "-lmlt",
                    "-Wl,-rpath," + PKG, "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("gpu_attn", [False, True])
def test_cpp_execute_matches_c_abi(demo, gpu_attn):
    out = subprocess.run([demo] + (["gpu-attn"] if gpu_attn else []), check=True, capture_output=True, text=True,
                         timeout=300).stdout
    r = json.loads(out.strip().splitlines()[-1])
    print("\n" + json.dumps(r))
    assert r["verify"] == "" and r["entries"] == r["tasks"] and r["makespan"] > 0
    assert r["steady_layer_time"] > 0 and 0 < r["gpu_util"] <= 1
    assert r["decode_layer"]["layer_total"] > 0 and r["decode_layer"]["gpu_ffn"] > 0
    assert r["err_layers"] == "invalid_argument" and r["err_kind"] in ("invalid_argument",
                                                                       "UnsupportedCombinationError")
    model = capi.ModelSpec(2, 1024, 3584, 8, 2, 8, 2, 2.0, 2.0)
    pol = capi.Policy(8, 4, int(gpu_attn), 1, 1.0 if gpu_attn else 0.25, 1.0 if gpu_attn else 0.0)
    tok = np.array([100 + 37 * i for i in range(8)], np.int32)
    ids = []
    for use_execute in (False, True):
        rt = Runtime(model, pol, budget_bytes=4e9, max_ctx=64)
        rt.prefill_synthetic(16, 9012)
        if use_execute:  # the C form of sim::execute on the reference DAG
            api = capi.load_product()
            hw = capi.HardwareSpec(4e9, 1e12, 6.5e12, 1.8e11, 5.5e10, 1.4e15, 2e12)
            dag = api.build_schedule(hw, model, capi.WorkloadSpec(16, 3), pol, "s4" if gpu_attn else "cgopipe",
                                     steps=3)
            d = rt.execute(dag, tok)
            with pytest.raises(capi.MltError):  # a DAG of another layer count does not match
                rt.execute(api.build_schedule(hw, model, capi.WorkloadSpec(16, 1), pol,
                                              "s4" if gpu_attn else "cgopipe", layers=3, steps=1), tok)
        else:
            d = rt.decode(tok, 3)
        assert d.report.timeline_ok == 1
        ids.append(d.ids.reshape(-1))
        rt.close()
    assert np.array_equal(ids[0], ids[1])
    assert np.array_equal(np.array(r["ids"], np.int32), ids[0])
