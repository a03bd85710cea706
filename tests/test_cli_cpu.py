"""The plan / latency commands over the reference's INI configs
(paper_2411_11217_b200/cli.py), mirroring the reference's CLI tests
(proj/tests/test_cli.cpp:58-203): hand-derived toy latency, plan = the
in-process search (here: the compiled reference's search_policy on the same
grid), exit codes 2 / 3, byte-identical artifacts across runs."""
import json
import subprocess
import sys

import pytest

from paper_2411_11217_b200 import capi
from test_config_parity import TOY

ROOT = __file__.rsplit("/tests/", 1)[0]


def run_cli(*args, cwd=ROOT):
    r = subprocess.run([sys.executable, "-m", "paper_2411_11217_b200", *args], cwd=cwd,
                       capture_output=True, text=True, timeout=120)
    return r.returncode, r.stdout, r.stderr


@pytest.fixture
def toy(tmp_path):
    p = tmp_path / "toy.cfg"
    p.write_text(TOY)
    return str(p)


def test_latency_toy_hand_numbers(toy, tmp_path):
    rc, _, err = run_cli("latency", "--config", toy, "--ctx", "10", "--out", str(tmp_path / "o"))
    assert rc == 0, err
    doc = json.loads((tmp_path / "o" / "latency.json").read_text())
    assert doc["latency"]["comm"] == 1792.0 and doc["latency"]["t_cpu"] == 256.0
    assert doc["latency"]["t_layer"] == 1792.0
    assert doc["policy"]["N"] == 8 and doc["policy"]["mu"] == 4
    assert doc["manifest"]["command"] == "latency" and doc["memory"]["feasible"] is True


def test_plan_toy_matches_reference_search(toy, tmp_path, ref):
    rc, _, err = run_cli("plan", "--config", toy, "--max-n-ub", "4", "--mu-list", "1,2,4,8",
                         "--out", str(tmp_path / "o"))
    assert rc == 0, err
    doc = json.loads((tmp_path / "o" / "plan.json").read_text())
    cfg = ref.parse_config(TOY)
    rw = [i * 0.05 for i in range(21)]
    grid = capi.make_grid([1, 2, 4, 8], [1, 2, 3, 4], rw, rw)
    exp = ref.search_policy(cfg.hardware, cfg.model, cfg.workload, grid)
    assert doc["policy"]["N"] == exp.policy.batch and doc["policy"]["mu"] == exp.policy.micro_batch
    assert doc["policy"]["r_w"] == exp.policy.weights_on_gpu
    assert doc["objective"] == pytest.approx(exp.objective, rel=1e-9)


def test_error_exit_codes(tmp_path, toy):
    assert run_cli("plan", "--config", "/nonexistent.cfg")[0] == 2
    assert run_cli("plan", "--config", toy, "--definitely-not-a-flag", "1")[0] == 2
    bad = tmp_path / "tiny.cfg"
    bad.write_text("[hardware]\nm_g = 10\nm_c = 10\nb_g = 50\nb_c = 10\nb_cg = 2\np_g = 100\n"
                   "p_c = 10\n[model]\nl = 2\nh1 = 8\nh2 = 16\nn_q = 4\nn_kv = 2\nn_e = 4\nk = 2\n"
                   "dt_w = 2\ndt_kv = 2\n[workload]\ns = 10\nn = 4\n")
    assert run_cli("plan", "--config", str(bad), "--max-n-ub", "2")[0] == 3
    rc, _, err = run_cli("latency", "--config", str(bad))
    assert rc == 2 and "[policy]" in err


def test_identical_runs_identical_artifacts(toy, tmp_path):
    outs = []
    for d in ("a", "b"):
        rc, _, err = run_cli("plan", "--config", toy, "--max-n-ub", "4", "--mu-list", "1,2,4,8",
                             "--out", str(tmp_path / d))
        assert rc == 0, err
        outs.append((tmp_path / d / "plan.json").read_bytes())
    assert outs[0] == outs[1]


def test_batch_command_matches_reference_batcher(tmp_path, ref):
    """`batch` (cli.cpp:398-442) on CSV and JSONL request files = the compiled
    reference's batch_requests on the same queue."""
    csv = tmp_path / "r.csv"
    csv.write_text("a,77\nb,418\n\nc,242\n  d,256\ne,1693\n")
    jl = tmp_path / "r.jsonl"
    jl.write_text('{"id": "j1", "input_len": 40}\n{"id": 7, "input_len": 90}\n')
    for path, reqs in ((csv, [("a", 77), ("b", 418), ("c", 242), ("d", 256), ("e", 1693)]),
                       (jl, [("j1", 40), ("7", 90)])):
        rc, _, err = run_cli("batch", "--requests", str(path), "--n-ub", "2", "--ubs", "2", "--gen-len", "8",
                             "--cache-size", "1200", "--out", str(tmp_path / "o"))
        assert rc == 0, err
        doc = json.loads((tmp_path / "o" / "batch.json").read_text())
        mbs, aborted = ref.batch_requests(reqs, 2, 2, 8, 1200, True)
        assert doc["micro_batches"] == mbs and doc["aborted"] == aborted
        lens = dict(reqs)
        assert doc["sums"] == [sum(lens[r] for r in mb) for mb in mbs]


def test_batch_command_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("a,77\nb;418\n")
    rc, _, err = run_cli("batch", "--requests", str(bad), "--n-ub", "2", "--ubs", "2", "--gen-len", "8",
                         "--cache-size", "1200")
    assert rc == 2 and "bad.csv:2" in err
    bad.write_text("a,7x\n")
    rc, _, err = run_cli("batch", "--requests", str(bad), "--n-ub", "2", "--ubs", "2", "--gen-len", "8",
                         "--cache-size", "1200")
    assert rc == 2 and "input_len must be an integer" in err
    assert run_cli("batch", "--requests", "/nonexistent", "--n-ub", "1", "--ubs", "1", "--gen-len", "1",
                   "--cache-size", "4")[0] == 2
    ok = tmp_path / "ok.csv"
    ok.write_text("a,7\n")
    rc, _, err = run_cli("batch", "--requests", str(ok), "--n-ub", "0", "--ubs", "1", "--gen-len", "1",
                         "--cache-size", "4")
    assert rc == 2  # InvalidBatchParametersError
