"""`run`: the plan -> execute loop on the GPU from an INI config
(paper_2411_11217_b200/cli.py): search on this machine's measured spec with
the config's m_g as the budget, execute the pick, report measured tok/s
against its HRM bound."""
import json
import subprocess
import sys

import pytest

ROOT = __file__.rsplit("/tests/", 1)[0]

SMALL = """[hardware]
m_g = 3G
m_c = 64G
b_g = 1000G
b_c = 100G
b_cg = 50G
p_g = 1000TFLOPS
p_c = 1TFLOPS
[model]
l = 2
h1 = 1024
h2 = 3584
n_q = 8
n_kv = 2
n_e = 8
k = 2
dt_w = 2
dt_kv = 2
[workload]
s = 48
n = 8
"""


@pytest.mark.gpu
def test_run_small_config(tmp_path):
    cfg = tmp_path / "small.cfg"
    cfg.write_text(SMALL)
    r = subprocess.run([sys.executable, "-m", "paper_2411_11217_b200", "run", "--config", str(cfg),
                        "--steps", "4", "--mu-list", "32,64", "--max-n-ub", "4", "--out", str(tmp_path / "o")],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    doc = json.loads((tmp_path / "o" / "run.json").read_text())
    print("\n[cli run]", json.dumps({k: doc[k] for k in ("policy", "throughput", "measured")}))
    assert doc["policy"]["F_g"] == 1
    assert doc["policy"]["A_g"] == 1 or doc["policy"]["N"] // doc["policy"]["mu"] >= 2
    m = doc["measured"]
    assert m["timeline_ok"] and m["decode_tok_s"] > 0 and m["steps"] == 4


SERVE = SMALL + """[policy]
N = 32
mu = 16
A_g = 0
F_g = 1
r_w = 0.5
r_c = 0
"""


@pytest.mark.gpu
def test_serve_ragged_requests(tmp_path):
    """`serve`: the reference batcher's variable-length micro-batches through GPU
    prefill + decode; every request served or aborted exactly once, gen_len ids
    each, deterministic across runs."""
    cfg = tmp_path / "serve.cfg"
    cfg.write_text(SERVE)
    lens = [5, 60, 17, 33, 8, 41, 29, 12, 55, 3, 47, 21, 38, 9, 26, 50, 14, 31, 44, 6, 19, 36, 52, 11,
            27, 2, 58, 23, 40, 16, 35, 7, 49, 30, 13, 45, 24, 39, 4, 200]
    req = tmp_path / "r.csv"
    req.write_text("".join(f"q{i},{n}\n" for i, n in enumerate(lens)))
    docs = []
    for k in range(2):
        r = subprocess.run([sys.executable, "-m", "paper_2411_11217_b200", "serve", "--config", str(cfg),
                            "--requests", str(req), "--max-ctx", "80", "--keep-outputs",
                            "--out", str(tmp_path / f"o{k}")], cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        docs.append(json.loads((tmp_path / f"o{k}" / "serve.json").read_text()))
    d = docs[0]
    print("\n[cli serve]", json.dumps({k: d[k] for k in ("served", "aborted", "batches", "tok_s", "decode_tok_s")}))
    assert d["aborted"] == ["q39"]  # 200 + 8 > max_ctx
    assert d["served"] == len(lens) - 1 and len(d["batches"]) == 2
    assert all(len(v) == 8 for v in d["outputs"].values())
    assert d["outputs"] == docs[1]["outputs"]
