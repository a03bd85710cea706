"""CGOPipe scheduler interface against the compiled reference.

Mirrors proj/tests/test_pipesim.cpp: the 8-unit hand trace (:53-84), the
page recipe (:97-116), S2/S3/S4 structure (:118-135), degenerate cases
(:137-176), placement errors (:192-211), determinism + replay equality
(:213-236), CGOPipe dominance (:238-255), the analytic steady-time bound
(:257-274) -- and additionally requires the product DAG to equal the
reference DAG task for task and edge for edge (issue order is the contract
the B200 executor follows).
"""
import random

import pytest

from paper_2411_11217_b200 import capi
from conftest import toy_hardware, toy_model, toy_policy, toy_workload


def hand_traced():
    d = capi.StepDurations()
    d.pre_attn, d.cpu_attn, d.post_attn = 1.0, 3.0, 1.0
    return d


def random_durations(rng):
    d = capi.StepDurations()
    d.pre_attn, d.cpu_attn, d.post_attn = (rng.uniform(0.1, 3.0) for _ in range(3))
    d.offload_qkv, d.load_hidden, d.weight_stage = (rng.uniform(0.01, 0.3) for _ in range(3))
    d.weight_upload = rng.uniform(0.5, 5.0)
    d.kv_load = rng.uniform(0.01, 0.3)
    d.gpu_attn = rng.uniform(0.1, 3.0)
    return d


def kinds(dag):
    return [capi.TASK_KINDS[t.kind] for t, _ in dag.tasks()]


def test_hand_trace_makespan_8(api, ref):
    dag = api.build_schedule_durations(hand_traced(), "cgopipe", 1, 1, 2)
    tl = dag.simulate()
    assert tl.makespan == 8.0
    assert dag.verify(tl) == ""
    m = dag.metrics(tl)
    assert abs(m.utilization[1] - 6.0 / 8.0) < 1e-12
    for (t, _), e in zip(dag.tasks(), tl.entries):
        k = capi.TASK_KINDS[t.kind]
        if k == "pre_attn":
            assert e.start == (0.0 if t.microbatch == 1 else 1.0)
        if k == "cpu_attn":
            assert e.start == (1.0 if t.microbatch == 1 else 4.0)
        if k == "post_attn":
            assert e.start == (4.0 if t.microbatch == 1 else 7.0)
    rdag = ref.build_schedule_durations(hand_traced(), "cgopipe", 1, 1, 2)
    assert rdag.dump() == dag.dump()
    replay = rdag.simulate("replay_simulate")
    assert [e.start for e in replay.entries] == [e.start for e in tl.entries]


def test_cgopipe_structure(api):
    ks = kinds(api.build_schedule_durations(hand_traced(), "cgopipe", 1, 1, 2))
    for k, n in (("pre_attn", 2), ("offload_qkv", 2), ("cpu_attn", 2), ("load_hidden", 2),
                 ("post_attn", 2), ("gpu_attn", 0), ("kv_load", 0)):
        assert ks.count(k) == n


def test_pages_one_per_microbatch(api):
    rng = random.Random(3)
    for n_ub in (1, 2, 4):
        d = random_durations(rng)
        dag = api.build_schedule_durations(d, "cgopipe", 3, 1, n_ub)
        pages = [t for t, _ in dag.tasks() if t.kind == 6 and t.layer == 2]
        assert len(pages) == n_ub
        assert all(1 <= t.page <= n_ub for t in pages)
        assert abs(sum(t.duration for t in pages) - d.weight_upload) <= 1e-12 * d.weight_upload


def test_s2_s3_s4_structure(api):
    rng = random.Random(5)
    ks = kinds(api.build_schedule_durations(random_durations(rng), "s4", 2, 1, 3))
    assert ks.count("kv_load") == 6 and ks.count("gpu_attn") == 6
    assert ks.count("cpu_attn") == 0 and ks.count("load_hidden") == 0
    for kind in ("s2", "s3"):
        ks = kinds(api.build_schedule_durations(random_durations(rng), kind, 3, 1, 4))
        assert ks.count("weight_to_gpu") == 3


def test_degenerate_cases(api):
    t = capi.Task(4, 1, 1, 0, 0, 0, 2.5, 0)
    dag = api.dag_from_tasks([(t, [])])
    assert dag.simulate().makespan == 2.5
    chain = capi.StepDurations()
    chain.pre_attn, chain.cpu_attn, chain.post_attn = 2.0, 3.0, 4.0
    assert api.build_schedule_durations(chain, "cgopipe", 1, 1, 1).simulate().makespan == 9.0
    z = api.build_schedule_durations(capi.StepDurations(), "cgopipe", 2, 1, 2)
    tl = z.simulate()
    assert tl.makespan == 0.0
    assert all(u == 0.0 for u in z.metrics(tl).utilization)


def test_errors(api):
    empty = api.dag_from_tasks([])
    with pytest.raises(capi.EmptyTimelineError):
        empty.metrics(capi.Timeline((capi.TimelineEntry * 1)(), 0.0, (capi.C.c_double * 5)()))
    a = capi.Task(0, 1, 1, 0, 0, 0, 1.0, 0)
    b = capi.Task(0, 1, 1, 0, 0, 0, 1.0, 0)
    cyc = api.dag_from_tasks([(a, [1]), (b, [0])])
    with pytest.raises(capi.CycleDetectedError):
        cyc.simulate()
    with pytest.raises(capi.MltError):
        api.build_schedule_durations(capi.StepDurations(), "cgopipe", 0, 1, 1)
    hw, m, w = toy_hardware(), toy_model(), toy_workload()
    p = toy_policy()
    p.attn_on_gpu = 1
    with pytest.raises(capi.UnsupportedCombinationError):
        api.build_schedule(hw, m, w, p, "cgopipe", 2, 1)
    with pytest.raises(capi.UnsupportedCombinationError):
        api.build_schedule(hw, m, w, toy_policy(), "s4", 2, 1)
    p = toy_policy()
    p.ffn_on_gpu = 0
    with pytest.raises(capi.UnsupportedCombinationError):
        api.build_schedule(hw, m, w, p, "cgopipe", 2, 1)


@pytest.mark.parametrize("kind", ["cgopipe", "s2", "s3", "s4"])
def test_dag_identical_to_reference_and_deterministic(api, ref, kind):
    rng = random.Random(11 + len(kind))
    for _ in range(25):
        layers, steps, ubs = rng.randint(1, 4), rng.randint(1, 3), rng.randint(1, 4)
        durs = [random_durations(rng) for _ in range(steps)]
        dag = api.build_schedule_durations(durs, kind, layers, steps, ubs)
        rdag = ref.build_schedule_durations(durs, kind, layers, steps, ubs)
        assert dag.dump() == rdag.dump()
        a, b, r = dag.simulate(), dag.simulate(), rdag.simulate()
        assert [(e.start, e.end) for e in a.entries] == [(e.start, e.end) for e in b.entries]
        assert [(e.start, e.end) for e in a.entries] == [(e.start, e.end) for e in r.entries]
        assert a.makespan == r.makespan and list(a.busy) == list(r.busy)
        assert dag.verify(a) == ""
        assert a.makespan >= max(a.busy) - 1e-9
        assert bytes(dag.metrics(a)) == bytes(rdag.metrics(r))
        assert dag.timeline_json(a, '{"m":1}') == rdag.timeline_json(r, '{"m":1}')


def test_cgopipe_dominates_unpaged(api):
    rng = random.Random(13)
    for _ in range(40):
        d = random_durations(rng)
        L, M = rng.randint(1, 4), rng.randint(1, 4)
        cgo = api.build_schedule_durations(d, "cgopipe", L, 1, M).simulate().makespan
        s2 = api.build_schedule_durations(d, "s2", L, 1, M).simulate().makespan
        s3 = api.build_schedule_durations(d, "s3", L, 1, M).simulate().makespan
        assert cgo <= s2 + 1e-9 and cgo <= s3 + 1e-9


def test_steady_layer_time_bound(api, ref):
    hw, m, w, p = toy_hardware(), toy_model(), toy_workload(), toy_policy()
    dag = api.build_schedule(hw, m, w, p, "cgopipe", 10, 1)
    assert dag.dump() == ref.build_schedule(hw, m, w, p, "cgopipe", 10, 1).dump()
    met = dag.metrics(dag.simulate())
    bound = api.layer_latency(hw, m, w, p, float(w.prompt_len + 1)).layer_total
    assert bound - 1e-9 <= met.steady_layer_time <= 1.25 * bound


def test_attention_grows_with_context(api):
    dag = api.build_schedule(toy_hardware(), toy_model(), toy_workload(), toy_policy(),
                             "cgopipe", 2, 2)
    cpu = {t.step: t.duration for t, _ in dag.tasks() if t.kind == 2}
    assert cpu[2] > cpu[1]


def test_mixtral_8x7b_task_count(api, ref):
    from conftest import mixtral_8x7b_model
    hw = capi.HardwareSpec(16e9, 196e9, 6548.5e9, 300e9, 55.5e9, 1393e12, 20e12)
    m, w = mixtral_8x7b_model(), capi.WorkloadSpec(512, 32)
    p = capi.Policy(256, 64, 0, 1, 0.10, 0.0)
    dag = api.build_schedule(hw, m, w, p, "cgopipe", 32, 1)
    assert len(dag) == 896
    assert dag.dump() == ref.build_schedule(hw, m, w, p, "cgopipe", 32, 1).dump()
