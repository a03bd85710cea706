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
