"""The graph the B200 executor runs (mlt_execution_dag), checked on CPU.

* same tasks and issue order as the reference DAG;
* PostAttn keeps every page gate of its layer (the expert FFN reads all
  experts); PreAttn keeps only pages holding QKV rows (none when QKV is
  resident); GpuAttn has none;
* write-after-read edges make the two-slot page pool safe: a page of global
  layer g+2 waits for every GPU task of layer g;
* the augmented graph is acyclic (simulate succeeds) and, with the
  reference's own analytic durations, data-exact gates close the per-layer
  link bubble of the reference gates: steady layer time within 0.5% of the
  HRM layer bound, versus ~2.6% above it with the reference gates.
"""
import pytest

from paper_2411_11217_b200 import capi
from conftest import mixtral_8x7b_model, toy_hardware, toy_model, toy_policy, toy_workload

B200 = capi.HardwareSpec(16e9, 196e9, 6548.5e9, 111e9, 55.6e9, 1393e12, 2e12)


def tasks_of(dag):
    return dag.tasks()


def test_same_issue_order_and_gates(api):
    m, w = mixtral_8x7b_model(), capi.WorkloadSpec(512, 32)
    p = capi.Policy(256, 64, 0, 1, 0.10, 0.0)
    ref = api.build_schedule(B200, m, w, p, "cgopipe", 4, 2)
    ex = api.execution_dag(ref, m, p, exact_gates=True)
    rt, et = tasks_of(ref), tasks_of(ex)
    assert len(rt) == len(et)
    for (a, _), (b, _) in zip(rt, et):
        assert (a.kind, a.step, a.layer, a.microbatch, a.page, a.resource) == \
            (b.kind, b.step, b.layer, b.microbatch, b.page, b.resource)
    L = 4
    up = {}
    for i, (t, _) in enumerate(et):
        if capi.TASK_KINDS[t.kind] == "weight_to_gpu":
            up.setdefault((t.step - 1) * L + t.layer, set()).add(i)
    for i, (t, deps) in enumerate(et):
        k = capi.TASK_KINDS[t.kind]
        g = (t.step - 1) * L + t.layer
        page_deps = {d for d in deps if capi.TASK_KINDS[et[d][0].kind] == "weight_to_gpu"}
        if k == "post_attn":
            assert up[g] <= page_deps  # all pages of its own layer
        if k == "pre_attn":
            assert not (page_deps & up[g])  # r_w=0.10: QKV is resident
        if k == "weight_to_gpu" and g > 2:
            gpu_g2 = {j for j, (u, _) in enumerate(et)
                      if capi.RESOURCES[u.resource] == "gpu" and (u.step - 1) * L + u.layer == g - 2}
            assert gpu_g2 <= set(deps)
    ex.simulate()  # acyclic


def test_streamed_qkv_is_gated_exactly(api):
    m, w = mixtral_8x7b_model(), capi.WorkloadSpec(512, 32)
    p = capi.Policy(256, 64, 0, 1, 0.0, 0.0)  # nothing resident: QKV rows head the blob (page 1)
    ref = api.build_schedule(B200, m, w, p, "cgopipe", 3, 1)
    et = tasks_of(api.execution_dag(ref, m, p))
    for t, deps in et:
        if capi.TASK_KINDS[t.kind] == "pre_attn":
            pages = [et[d][0].page for d in deps if capi.TASK_KINDS[et[d][0].kind] == "weight_to_gpu"]
            assert pages == [1]


def test_reference_gates_mode_keeps_reference_edges(api):
    hw, m, w, p = toy_hardware(), toy_model(), toy_workload(), toy_policy()
    m.hidden_dim, m.ffn_dim, m.q_heads, m.kv_heads = 256, 256, 2, 1  # 128-row blocks
    ref = api.build_schedule(hw, m, w, p, "cgopipe", 3, 2)
    ex = api.execution_dag(ref, m, p, exact_gates=False)
    for (a, da), (b, db) in zip(tasks_of(ref), tasks_of(ex)):
        assert set(da) <= set(db)


@pytest.mark.parametrize("mu", [64, 128])
def test_exact_gates_close_the_link_bubble_in_the_model(api, mu):
    m, w = mixtral_8x7b_model(), capi.WorkloadSpec(512, 32)
    p = capi.Policy(256, mu, 0, 1, 0.10, 0.0)
    ref = api.build_schedule(B200, m, w, p, "cgopipe", 32, 1)
    bound = api.layer_latency(B200, m, w, p, 513.0).layer_total
    sim_ref = ref.metrics(ref.simulate()).steady_layer_time
    ex = api.execution_dag(ref, m, p, exact_gates=True)
    sim_ex = ex.metrics(ex.simulate()).steady_layer_time
    assert sim_ref > 1.01 * bound          # the reference schedule's own bubble
    assert sim_ex <= 1.005 * bound          # gone with data-exact gates
    assert sim_ex >= bound * (1 - 1e-9)     # never beats the link bound
