"""Policy search (§8(f) rank 3) and request batcher (§8(f) rank 2) against the
compiled reference.

search_policy: the product's OpenMP search (csrc/plan/search.cpp) must return
the same PlanResult, bit for bit, as the reference's search
(proj/src/planner.cpp search_policy) and the same winner as the reference's
serial brute force (proj/tests/support/search_reference.cpp), mirroring
proj/tests/test_planner.cpp:214-325.

batch_requests: Algorithm 2 (proj/src/batcher.cpp) — identical micro-batch
memberships, orders and abort lists to the reference's batcher and, with
flushing off, to its literal replay (proj/tests/support/batch_reference.cpp),
mirroring proj/tests/test_batcher.cpp:46-200.
"""
import random

import pytest

from paper_2411_11217_b200 import capi
from conftest import mixtral_8x7b_model, toy_hardware, toy_model, toy_workload


def plan_tuple(r):
    p, b, m = r.policy, r.breakdown, r.memory
    return ((p.batch, p.micro_batch, p.attn_on_gpu, p.ffn_on_gpu, p.weights_on_gpu, p.kv_on_gpu),
            tuple(getattr(b, f) for f, _ in b._fields_),
            (m.gpu_bytes, m.cpu_bytes, m.feasible),
            r.decode_throughput, r.generation_throughput, r.objective)


def pol_tuple(p):
    return (p.batch, p.micro_batch, p.attn_on_gpu, p.ffn_on_gpu, p.weights_on_gpu, p.kv_on_gpu)


def random_scenario(rng):
    """test_planner.cpp:22-52: physically ordered specs whose memory limits
    leave part of the grid feasible."""
    small = lambda: rng.randint(1, 6)  # noqa: E731
    mag = lambda: rng.uniform(1.0, 50.0)  # noqa: E731
    kvh = small()
    qh = kvh * small()
    hidden = qh * 2 * small()
    experts = 1 + small()
    top_k = 1 + (small() - 1) % experts
    m = capi.ModelSpec(2 + small(), hidden, hidden * 2, qh, kvh, experts, top_k, 2.0, 2.0)
    w = capi.WorkloadSpec(8 * small(), 2 * small())
    cpu_bw = mag()
    gpu_bw = cpu_bw * (1 + mag())
    link_bw = cpu_bw / (1 + mag() / 10)
    cpu_flops = mag()
    gpu_flops = cpu_flops * (1 + mag())
    hw = capi.HardwareSpec(0, 0, gpu_bw, cpu_bw, link_bw, gpu_flops, cpu_flops)
    return hw, m, w


def finish_memory(api, rng, hw, m, w):
    wt, kv = api.memory_totals(m, w, 64)
    hw.gpu_mem_bytes = rng.uniform(0.2, 2.0) * wt + 4096
    hw.cpu_mem_bytes = (1.5 + rng.uniform(1.0, 50.0) / 10) * (wt + kv)


def small_grid(rng):
    mu = [v for v in (1, 2, 4, 8, 16) if rng.randint(0, 4) < 3] or [1, 4]
    return capi.make_grid(mu, [1, 2, 3, 4], [0.0, 0.25, 0.5, 0.75, 1.0], [0.0, 0.5, 1.0])


def brute(ref, hw, m, w, grid):
    pol, obj = capi.Policy(), capi.C.c_double()
    found = ref.check(ref.fn["brute_force_search"](capi.C.byref(hw), capi.C.byref(m), capi.C.byref(w),
                                                   capi.C.byref(grid), capi.C.byref(pol),
                                                   capi.C.byref(obj)))
    return (pol, obj.value) if found else None


def test_default_grid_candidate_count(api, ref):
    # SearchGrid::defaults(): the grid the CLI searches (planner.hpp:77-100)
    assert api.search_candidate_count() == ref.search_candidate_count()
    assert api.search_candidate_count() == 2010624
    g = capi.make_grid([4], [2], [0.0], [0.0], [0], [1])
    assert api.search_candidate_count(g) == 1


def test_single_feasible_policy(api, ref):
    # test_planner.cpp:234-248
    g = capi.make_grid([4], [2], [0.0], [0.0], [0], [1])
    r = api.search_policy(toy_hardware(), toy_model(), toy_workload(), g)
    assert (r.policy.batch, r.policy.micro_batch) == (8, 4)
    assert plan_tuple(r) == plan_tuple(ref.search_policy(toy_hardware(), toy_model(), toy_workload(), g))


def test_memory_pressure_forces_offload(api, ref):
    # test_planner.cpp:250-265
    m = toy_model()
    m.layers = 4
    hw = toy_hardware()
    hw.gpu_mem_bytes = 10000
    g = capi.make_grid([1, 2, 4], [1, 2], [0.0, 0.5, 1.0], [0.0], [0], [1])
    r = api.search_policy(hw, m, toy_workload(), g)
    assert r.policy.weights_on_gpu < 1.0
    assert plan_tuple(r) == plan_tuple(ref.search_policy(hw, m, toy_workload(), g))


def test_no_feasible_policy_names_tightest_constraint(api, ref):
    # test_planner.cpp:267-281
    hw = toy_hardware()
    hw.gpu_mem_bytes = hw.cpu_mem_bytes = 10
    g = capi.make_grid([1], [1], [0.0], [0.0], [0], [1])
    with pytest.raises(capi.NoFeasiblePolicyError) as e:
        api.search_policy(hw, toy_model(), toy_workload(), g)
    assert "tightest violated constraint" in str(e.value)
    with pytest.raises(capi.NoFeasiblePolicyError) as e2:
        ref.search_policy(hw, toy_model(), toy_workload(), g)
    assert api.error() == ref.error() or str(e.value).split(":", 1)[-1] == str(e2.value).split(":", 1)[-1]


@pytest.mark.parametrize("seed", [31, 32, 33])
def test_random_grids_match_reference_and_brute_force(api, ref, seed):
    # test_planner.cpp:214-232, plus bitwise equality with the reference search
    rng = random.Random(seed)
    compared = 0
    for _ in range(10):
        hw, m, w = random_scenario(rng)
        finish_memory(api, rng, hw, m, w)
        g = small_grid(rng)
        b = brute(ref, hw, m, w, g)
        if b is None:
            with pytest.raises(capi.NoFeasiblePolicyError):
                api.search_policy(hw, m, w, g)
            with pytest.raises(capi.NoFeasiblePolicyError):
                ref.search_policy(hw, m, w, g)
            continue
        for objective in (0, 1):
            r = api.search_policy(hw, m, w, g, objective)
            assert plan_tuple(r) == plan_tuple(ref.search_policy(hw, m, w, g, objective))
        r = api.search_policy(hw, m, w, g)
        assert r.objective == b[1] and pol_tuple(r.policy) == pol_tuple(b[0])
        compared += 1
    assert compared > 0


def test_improving_hardware_never_worsens(api):
    # test_planner.cpp:283-309
    rng = random.Random(41)
    compared = 0
    for _ in range(12):
        hw, m, w = random_scenario(rng)
        finish_memory(api, rng, hw, m, w)
        g = small_grid(rng)
        try:
            base = api.search_policy(hw, m, w, g)
        except capi.NoFeasiblePolicyError:
            continue
        compared += 1
        for f, _ in capi.HardwareSpec._fields_:
            better = capi.HardwareSpec(*[getattr(hw, n) for n, _ in capi.HardwareSpec._fields_])
            setattr(better, f, getattr(hw, f) * 2)
            if api.validate(hw=better):
                continue
            assert api.search_policy(better, m, w, g).objective <= base.objective + 1e-15
    assert compared > 0


def test_b200_default_grid_mixtral_8x7b(api, ref):
    """The full default grid (2,010,624 candidates) on the headline setting:
    Mixtral-8x7B, 16 GB B200 budget, prompt 512, gen 32 — identical plan."""
    hw = capi.HardwareSpec(16e9, 196e9, 6548.5e9, 111e9, 55.6e9, 1393e12, 2e12)
    m, w = mixtral_8x7b_model(), capi.WorkloadSpec(512, 32)
    r = api.search_policy(hw, m, w)
    assert plan_tuple(r) == plan_tuple(ref.search_policy(hw, m, w))
    assert r.memory.feasible and r.memory.gpu_bytes <= hw.gpu_mem_bytes
    # ctx override and latency objective take the same path in both builds
    for obj, ctx in ((1, -1.0), (0, 4096.0)):
        assert plan_tuple(api.search_policy(hw, m, w, None, obj, ctx)) == \
            plan_tuple(ref.search_policy(hw, m, w, None, obj, ctx))


# ---------------------------------------------------------------- batcher --
def queue(lengths, prefix="r"):
    return [(f"{prefix}{i}", n) for i, n in enumerate(lengths)]


def lens_of(q, ids):
    d = dict(q)
    return [d[i] for i in ids]


def test_batcher_hand_trace(api, ref):
    # test_batcher.cpp:46-57
    q = queue([10, 8, 5, 3])
    mbs, ab = api.batch_requests(q, 2, 2, 1, 1000)
    assert [lens_of(q, mb) for mb in mbs] == [[8, 5], [10, 3]] and ab == []
    assert (mbs, ab) == ref.batch_requests(q, 2, 2, 1, 1000)


def test_batcher_empty_queue(api):
    assert api.batch_requests([], 2, 2, 1, 100) == ([], [])


def test_batcher_budget_guard(api, ref):
    # test_batcher.cpp:70-88
    q = queue([12, 10, 4])
    mbs, ab = api.batch_requests(q, 2, 2, 5, 20)
    assert lens_of(q, ab) == [4] and [len(mb) for mb in mbs] == [1, 1]
    lit = api.batch_requests(q, 2, 2, 5, 20, flush_partials=False)
    assert lit[0] == [] and len(lit[1]) == 1
    assert (mbs, ab) == ref.batch_requests(q, 2, 2, 5, 20)
    assert lit == ref.batch_requests(q, 2, 2, 5, 20, flush_partials=False)


def test_batcher_exhausted_partitions(api):
    # test_batcher.cpp:90-100
    q = queue([5, 4, 3])
    mbs, ab = api.batch_requests(q, 1, 1, 1, 100)
    assert [lens_of(q, mb) for mb in mbs] == [[5]] and len(ab) == 2


def test_batcher_invalid_parameters(api):
    # test_batcher.cpp:102-111
    with pytest.raises(capi.MltError):
        api.batch_requests([], 0, 1, 1, 100)
    with pytest.raises(capi.MltError):
        api.batch_requests([], 1, 1, 1, 1)
    with pytest.raises(capi.MltError):
        api.batch_requests([("bad", 0)], 1, 1, 1, 100)


def test_batcher_random_queues_match_reference_and_replay(api, ref):
    # test_batcher.cpp:113-146 plus bitwise equality with the reference batcher
    rng = random.Random(17)
    for _ in range(150):
        q = [(f"q{i}", rng.randint(1, 4096)) for i in range(rng.randint(0, 200))]
        n_ub, ubs, gen = rng.randint(1, 8), rng.randint(1, 64), rng.randint(1, 64)
        cache = gen + 1 + rng.randint(1, 4096) * 2
        for flush in (False, True):
            got = api.batch_requests(q, n_ub, ubs, gen, cache, flush)
            assert got == ref.batch_requests(q, n_ub, ubs, gen, cache, flush)
        lit = api.batch_requests(q, n_ub, ubs, gen, cache, False)
        assert lit == ref.batch_requests(q, n_ub, ubs, gen, cache, False, fn="replay_batching")
        for mb in lit[0]:
            assert sum(lens_of(q, mb)) + len(mb) * gen <= cache


def test_batcher_order_invariance(api):
    # test_batcher.cpp:148-171
    rng = random.Random(19)
    q = queue([64, 64, 32, 32, 16, 16, 8, 8, 4, 4])

    def sums(qq):
        return sorted(sum(lens_of(qq, mb)) for mb in api.batch_requests(qq, 3, 3, 2, 500)[0])

    base = sums(q)
    for _ in range(20):
        rng.shuffle(q)
        assert sums(q) == base
