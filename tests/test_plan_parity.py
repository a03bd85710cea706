"""The B200 build's cost model / planner against the compiled reference.

Golden numbers are the reference's own known-answer tests
(proj/tests/test_opcost.cpp:30-137, test_planner.cpp:78-178); every other
check compares product (mlt_*) and reference (ref_*) bit for bit on random
specs, mirroring test_planner.cpp's seeded property tests.
"""
import random

import pytest

from paper_2411_11217_b200 import capi
from conftest import (mixtral_8x7b_model, mixtral_8x22b_model, toy_hardware, toy_model,
                      toy_policy, toy_workload)


def test_toy_opcost_hand_counts(api):
    m = toy_model()
    p1 = api.op_profiles(m, 1, 10)
    assert p1["attention"].flops == 320.0 and p1["attention"].cpu_bytes == 160.0
    p2 = api.op_profiles(m, 2, 10)
    assert p2["attention"].flops == 640.0 and p2["attention"].cpu_bytes == 320.0
    f = api.op_profiles(m, 1, 10, 0.0)["ffn"]
    assert f.flops == 1536.0 and f.link_bytes == 3072.0
    assert api.op_profiles(m, 1, 10, 1.0)["ffn"].link_bytes == 0.0
    p = api.op_profiles(m, 1, 10)
    assert p["qkv"].flops == 256.0 and p["output"].flops == 128.0
    assert p["qkv"].gpu_bytes == 256.0 and p["output"].gpu_bytes == 128.0
    assert api.layer_weight_bytes(m).total() == 3520.0
    pol = toy_policy()
    t = api.transfer_sizes(m, pol, 10)
    assert (t.weight_stream, t.hidden_upload, t.kv_upload) == (3520.0, 64.0, 0.0)
    pol.attn_on_gpu, pol.kv_on_gpu = 1, 0.5
    assert api.transfer_sizes(m, pol, 10).kv_upload == 0.5 * 4 * 2 * 10 * 2 * 2 * 2
    assert api.memory_totals(m, toy_workload(), 8) == (7040.0, 3584.0)


def test_mixtral_8x22b_expert_bytes_exact(api):
    m = mixtral_8x22b_model()
    assert m.layers * api.layer_weight_bytes(m).experts == 270582939648.0


def test_toy_breakdown_golden(api, ref):
    lat = api.layer_latency(toy_hardware(), toy_model(), toy_workload(), toy_policy(), 10.0)
    assert lat.link_upload == 1792.0
    assert lat.cpu_attention == 256.0 and lat.cpu_ffn == 0.0
    assert abs(lat.gpu_total() - 153.6) < 1e-12 * 153.6
    assert lat.layer_total == 1792.0
    o = (capi.C.c_double * 5)()
    ref.check(ref.fn["oracle_layer_latency"](capi.C.byref(toy_hardware()),
                                             capi.C.byref(toy_model()),
                                             capi.C.byref(toy_policy()), 10.0, o))
    assert (lat.link_upload, lat.cpu_attention, lat.gpu_total(), lat.layer_total) == \
        (o[0], o[1], o[3], o[4])


def test_footprint_hand_counts(api):
    hw, m, w = toy_hardware(), toy_model(), toy_workload()
    res = capi.Policy(8, 1, 1, 1, 1.0, 1.0)
    assert api.memory_footprint(hw, m, w, res).cpu_bytes == 0.0
    assert api.memory_footprint(hw, m, w, toy_policy()).cpu_bytes == 7040.0 + 3584.0 + 2 * 3520.0


def test_tp_rules(api):
    hw = toy_hardware()
    d = api.apply_tensor_parallelism(hw, 2)
    assert (d.gpu_mem_bytes, d.gpu_bw, d.gpu_flops, d.cpu_bw, d.link_bw) == \
        (2e6, 100.0, 200.0, 10.0, 2.0)
    b = api.apply_tensor_parallelism(hw, 4, b200_rule=True, host_read_cap=5.0)
    assert b.link_bw == 5.0 and b.gpu_flops == 400.0
    with pytest.raises(capi.MltError):
        api.apply_tensor_parallelism(hw, 0)


def test_infeasible_policy_raises(api):
    hw = toy_hardware()
    hw.gpu_mem_bytes = 1.0
    with pytest.raises(capi.InfeasiblePolicyError):
        api.layer_latency(hw, toy_model(), toy_workload(), capi.Policy(8, 4, 1, 1, 1.0, 1.0), 10)


def _random_case(rng):
    heads = rng.choice([1, 2, 4, 8])
    n_kv = rng.choice([d for d in (1, 2, 4, 8) if heads % d == 0])
    m = capi.ModelSpec(rng.randint(1, 8), heads * rng.randint(1, 64), 2 * rng.randint(1, 512),
                       heads, n_kv, rng.randint(1, 16), 1, 2.0, rng.choice([1.0, 2.0]))
    m.top_k = rng.randint(1, m.experts)
    hw = capi.HardwareSpec(10 ** rng.uniform(4, 12), 10 ** rng.uniform(6, 13),
                           10 ** rng.uniform(2, 12), 10 ** rng.uniform(1, 11),
                           10 ** rng.uniform(0, 10), 10 ** rng.uniform(3, 15),
                           10 ** rng.uniform(2, 12))
    mu = rng.choice([1, 2, 4, 8, 16, 64])
    pol = capi.Policy(mu * rng.randint(1, 8), mu, rng.randint(0, 1), rng.randint(0, 1),
                      rng.choice([0.0, 0.05, 0.1, 0.35, 0.9, 1.0]), 0.0)
    if pol.attn_on_gpu:
        pol.kv_on_gpu = rng.choice([0.0, 0.5, 1.0])
    w = capi.WorkloadSpec(rng.randint(1, 600), rng.randint(1, 40))
    return hw, m, w, pol


def test_planner_matches_reference_bitwise(api, ref):
    rng = random.Random(23)
    compared = 0
    for _ in range(400):
        hw, m, w, pol = _random_case(rng)
        ctx = float(rng.randint(1, 700))
        for name in ("attention", "ffn", "qkv", "output"):
            a = api.op_profiles(m, pol.micro_batch, ctx, pol.weights_on_gpu)[name]
            b = ref.op_profiles(m, pol.micro_batch, ctx, pol.weights_on_gpu)[name]
            assert bytes(a) == bytes(b), name
        assert bytes(api.transfer_sizes(m, pol, ctx)) == bytes(ref.transfer_sizes(m, pol, ctx))
        assert bytes(api.memory_footprint(hw, m, w, pol)) == \
            bytes(ref.memory_footprint(hw, m, w, pol))
        try:
            b = ref.layer_latency(hw, m, w, pol, ctx)
        except capi.InfeasiblePolicyError:
            with pytest.raises(capi.InfeasiblePolicyError):
                api.layer_latency(hw, m, w, pol, ctx)
            continue
        assert bytes(api.layer_latency(hw, m, w, pol, ctx)) == bytes(b)
        assert bytes(api.estimate_throughput(hw, m, w, pol)) == \
            bytes(ref.estimate_throughput(hw, m, w, pol))
        compared += 1
    assert compared > 50


def test_b200_headline_bound_matches_reference(api, ref):
    """The headline HRM bound computed both ways."""
    hw = capi.HardwareSpec(16e9, 196e9, 6548.5e9, 300e9, 55.5e9, 1393e12, 20e12)
    m, w = mixtral_8x7b_model(), capi.WorkloadSpec(512, 32)
    for mu in (64, 256):
        pol = capi.Policy(256, mu, 0, 1, 0.10, 0.0)
        a, b = api.estimate_throughput(hw, m, w, pol), ref.estimate_throughput(hw, m, w, pol)
        assert bytes(a) == bytes(b)
        assert 150 < a.decode_throughput < 190


def test_b200_hrm_nvlink_roof(api):
    """estimate_throughput_b200: tp=1 is estimate_throughput bit for bit; at tp>1
    every layer's GPU FFN term grows by exactly the NVLink all-reduce time
    (2 fp32 [mu, h1] all-reduces per micro-batch, ring 2(tp-1)/tp)."""
    m = mixtral_8x22b_model()
    w = capi.WorkloadSpec(512, 32)
    p = capi.Policy(256, 64, 0, 1, 0.15, 0.0)
    hw = capi.HardwareSpec(16e9, 1e13, 6.5e12, 1.1e11, 5.56e10, 1.39e15, 2e12)
    big = capi.HardwareSpec(80e9, 1e13, 6.5e12, 1.1e11, 5.56e10, 1.39e15, 2e12)
    a = api.estimate_throughput(big, m, w, p)
    b = api.estimate_throughput_b200(big, m, w, p, 1, 900e9)
    assert a.decode_throughput == b.decode_throughput and a.breakdown.gpu_ffn == b.breakdown.gpu_ffn
    tp = 4
    hw4 = api.apply_tensor_parallelism(hw, tp, b200_rule=True, host_read_cap=0.0)
    base = api.estimate_throughput(hw4, m, w, p)
    ext = api.estimate_throughput_b200(hw4, m, w, p, tp, 900e9)
    t_nvl = 4 * 2 * (2 * 3 / 4) * 64 * 6144 * 4 / 900e9
    assert abs((ext.breakdown.gpu_ffn - base.breakdown.gpu_ffn) - t_nvl) < 1e-15
    assert ext.decode_throughput <= base.decode_throughput
    # link-bound here: the NVLink roof does not move the bound
    assert ext.breakdown.layer_total == base.breakdown.layer_total
