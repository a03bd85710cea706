"""Hierarchical roofline (lightplan/hrm.hpp) against the compiled reference.

Known answers are the reference's own (proj/tests/test_hrm.cpp:29-128); the
rest compares product (mlt_*) and reference (ref_*) bit for bit on random
specs drawn like test_hrm.cpp's random_hw (:13-24)."""
import math
import random

import pytest

from paper_2411_11217_b200 import capi
from conftest import mixtral_8x7b_model, toy_hardware, toy_model

GPU, CPU = capi.LEVEL_GPU, capi.LEVEL_CPU


def random_hw(rng):
    """test_hrm.cpp:13-24: magnitudes in [0.1, 1000), GPU >= CPU."""
    mag = lambda: rng.uniform(0.1, 1000.0)  # noqa: E731
    cpu_bw = mag()
    gpu_bw = cpu_bw * (1.0 + mag())
    link = mag()
    cpu_f = mag()
    gpu_f = cpu_f * (1.0 + mag())
    return capi.HardwareSpec(1e9, 1e9, gpu_bw, cpu_bw, link, gpu_f, cpu_f)


def test_toy_known_answers(api):
    hw = toy_hardware()
    # test_hrm.cpp:29-34
    assert api.attainable_local(GPU, 1.0, hw) == 50.0
    assert api.attainable_local(GPU, 4.0, hw) == 100.0
    assert api.attainable_local(CPU, 0.0, hw) == 0.0
    # :36-42
    assert api.attainable_cross(4.0, 2.0, hw) == 4.0
    assert api.attainable_cross(0.0, 0.0, hw) == 0.0
    assert api.attainable_cross(4.0, math.inf, hw) == api.attainable_local(GPU, 4.0, hw)
    # :62-74
    assert api.turning_point_p1(2.0, hw) == 5.0
    assert api.turning_point_p1(0.5, hw) == 2.5
    assert api.turning_point_p2(4.0, hw) == 50.0
    assert api.turning_point_p2(1.0, hw) == 25.0
    fast = toy_hardware()
    fast.link_bw = fast.cpu_bw
    fast.cpu_flops = fast.gpu_flops = 1e18
    assert api.turning_point_p1(3.0, fast) == 3.0
    # :93-98
    assert api.balance_gap(1.0, 25.0, hw) == 0.0
    assert api.balance_gap(1.0, 10.0, hw) == 30.0
    assert api.balance_gap(0.0, 0.0, hw) == 0.0


def test_cross_bounded_and_monotone():
    """test_hrm.cpp:44-59 over 2000 seeded specs (product only: a property)."""
    api = capi.load_product()
    rng = random.Random(3)
    for _ in range(2000):
        h = random_hw(rng)
        gi, ci = rng.uniform(0, 100), rng.uniform(0, 100)
        b = api.attainable_cross(gi, ci, h)
        assert b <= h.gpu_flops and b <= h.gpu_bw * gi and b <= h.link_bw * ci
        assert api.attainable_cross(gi * 1.5, ci, h) >= b
        assert api.attainable_cross(gi, ci * 1.5, h) >= b


def test_cross_at_p1_recovers_cpu_local(api):
    """test_hrm.cpp:77-91."""
    rng = random.Random(5)
    for _ in range(2000):
        hw = random_hw(rng)
        ci = rng.uniform(0.01, 50.0)
        p1 = api.turning_point_p1(ci, hw)
        local = api.attainable_local(CPU, ci, hw)
        unb = capi.HardwareSpec(hw.gpu_mem_bytes, hw.cpu_mem_bytes, 1e30, hw.cpu_bw, hw.link_bw, 1e30,
                                hw.cpu_flops)
        assert api.attainable_cross(1e20, p1, unb) == pytest.approx(local, rel=1e-12)


def test_bitwise_vs_reference_random(api, ref):
    rng = random.Random(11)
    for _ in range(3000):
        hw = random_hw(rng)
        gi, ci = rng.uniform(0, 500), rng.uniform(0, 500)
        for lv in (GPU, CPU):
            assert api.attainable_local(lv, gi, hw) == ref.attainable_local(lv, gi, hw)
        assert api.attainable_cross(gi, ci, hw) == ref.attainable_cross(gi, ci, hw)
        assert api.turning_point_p1(ci, hw) == ref.turning_point_p1(ci, hw)
        assert api.turning_point_p2(gi, hw) == ref.turning_point_p2(gi, hw)
        assert api.balance_gap(gi, ci, hw) == ref.balance_gap(gi, ci, hw)


def test_roofline_series_csv_matches_reference(api, ref):
    """test_hrm.cpp:100-128 (op points, link roof slope, header) + the CSV
    byte for byte against the reference on toy and 8x7B/B200 inputs."""
    hw = toy_hardware()
    m = toy_model()
    pr = api.op_profiles(m, 4, 10, 0.0)
    profiles, names = [pr["ffn"], pr["attention"]], ["ffn_mu4", "attn_mu4"]
    csv = api.roofline_csv(profiles, names, hw)
    assert csv == ref.roofline_csv(profiles, names, hw)
    rows = [r.split(",") for r in csv.strip().split("\n")[1:]]
    ops = [r for r in rows if r[1] == "op_point"]
    assert len(ops) == 4
    link = [r for r in rows if r[1] == "mem_ji"]
    assert link and all(float(r[3]) / float(r[2]) == pytest.approx(hw.link_bw) for r in link)
    assert pr["ffn"].link_bytes and pr["ffn"].flops / pr["ffn"].link_bytes < api.turning_point_p2(4.0, hw)
    assert csv.startswith("series,kind,intensity,bound\n") and "ffn_mu4@gpu,op_point," in csv
    with pytest.raises(capi.MltError):
        api.roofline_csv([], [], hw)
    # B200 spec, 8x7B decode operators at mu=64 / ctx 528, non-default grids
    b200 = capi.HardwareSpec(16e9, 196e9, 6554.2e9, 178.5e9, 55.5e9, 1393e12, 2e12)
    pr = api.op_profiles(mixtral_8x7b_model(), 64, 528, 0.10)
    profs = [pr[k] for k in ("attention", "ffn", "qkv", "output")]
    nm = ["attention", "ffn", "qkv", "output"]
    for g in (None, capi.RooflineGrid(1e-3, 1e5, 16), capi.RooflineGrid(0.5, 0.5, 64),
              capi.RooflineGrid(1.0, 10.0, 1)):
        assert api.roofline_csv(profs, nm, b200, g) == ref.roofline_csv(profs, nm, b200, g)


def test_b200_turning_points_8x7b(api):
    """SURVEY §8(a) a13 on the B200 spec: ridge p_g/b_g ~ 213 FLOP/B; the 8x7B
    expert FFN at mu=64 sits far left of P2, i.e. link-bound when paged."""
    b200 = capi.HardwareSpec(16e9, 196e9, 6548.5e9, 300e9, 55e9, 1393e12, 20e12)
    assert b200.gpu_flops / b200.gpu_bw == pytest.approx(212.7, rel=1e-3)
    ffn = api.op_profiles(mixtral_8x7b_model(), 64, 528, 0.10)["ffn"]
    p2 = api.turning_point_p2(ffn.gpu_intensity() if hasattr(ffn, "gpu_intensity") else
                              ffn.flops / ffn.gpu_bytes, b200)
    assert ffn.flops / ffn.link_bytes < p2
    assert api.attainable_cross(ffn.flops / ffn.gpu_bytes, ffn.flops / ffn.link_bytes, b200) == \
        pytest.approx(b200.link_bw * ffn.flops / ffn.link_bytes)
