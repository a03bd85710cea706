"""INI config surface (include/lightplan/config.hpp, csrc/plan/config.cpp)
against the compiled reference parser (oracle/_ref, config.cpp:148-426).

Known answers mirror the reference's own test_config.cpp:100-172 (unit
suffixes, FLOP suffixes, unknown keys / missing sections with their lines,
validation issues, bit-exact round trip, duplicate keys); a seeded mutation
fuzz then compares product and reference outcome by outcome: the parsed
fields bit for bit, or the same error line and message."""
import random

import pytest

from paper_2411_11217_b200 import capi

TOY = """# toy fixture: hand-checkable units
[hardware]
m_g = 1M
m_c = 1M
b_g = 50
b_c = 10
b_cg = 2
p_g = 100
p_c = 10

[model]
l = 2
h1 = 8
h2 = 16
n_q = 4
n_kv = 2
n_e = 4
k = 2
dt_w = 2
dt_kv = 2

[workload]
s = 10
n = 4

[policy]
N = 8
mu = 4
A_g = 0
F_g = 1
r_w = 0
r_c = 0
"""

B200 = """# Mixtral-8x7B on one B200 (measured link / host numbers, 16 GB budget)
[hardware]
m_g = 16G      # budget
m_c = 196G
b_g = 6548.5G
b_c = 174.2g
b_cg = 55.6G
p_g = 1393TFLOPS
p_c = 2tflops
[model]
l = 32
h1 = 4096
h2 = 14336
n_q = 32
n_kv = 8
n_e = 8
k = 2
dt_w = 1.517578125
dt_kv = 2
[workload]
s = 512
n = 32
"""


def outcome(api, text):
    try:
        c = api.parse_config(text)
    except capi.ConfigError as e:
        return ("error", e.line, e.message)
    fields = []
    for part in ("hardware", "model", "workload", "policy"):
        s = getattr(c, part)
        fields += [(part, n, repr(getattr(s, n))) for n, _ in s._fields_]
    return ("ok", c.has_policy, tuple(fields), api.serialize_config(c))


def test_unit_suffixes(api):
    c = api.parse_config(TOY)
    assert c.hardware.gpu_mem_bytes == 1e6 and c.hardware.link_bw == 2.0
    assert c.model.ffn_dim == 16 and c.workload.prompt_len == 10
    assert c.has_policy and c.policy.batch == 8 and not c.policy.attn_on_gpu


def test_flops_suffixes(api):
    c = api.parse_config(
        "[hardware]\nm_g = 16G\nm_c = 192G\nb_g = 300G\nb_c = 50G\nb_cg = 8G\n"
        "p_g = 65TFLOPS\np_c = 750GFLOPS\n"
        "[model]\nl = 2\nh1 = 8\nh2 = 16\nn_q = 4\nn_kv = 2\nn_e = 4\nk = 2\ndt_w = 2\ndt_kv = 2\n"
        "[workload]\ns = 10\nn = 4\n")
    assert c.hardware.link_bw == 8e9 and c.hardware.gpu_flops == 65e12 and c.hardware.cpu_flops == 750e9
    assert not c.has_policy


def test_unknown_key_and_missing_section(api):
    with pytest.raises(capi.ConfigError) as e:
        api.parse_config("[hardware]\nm_g = 1\nnope = 3\n")
    assert e.value.line == 3
    with pytest.raises(capi.ConfigError) as e:
        api.parse_config("[hardware]\nm_g = 1\n")
    assert "missing" in e.value.message


def test_validation_issues_surface(api):
    with pytest.raises(capi.ConfigError) as e:
        api.parse_config(TOY.replace("n_q = 4", "n_q = 6").replace("n_kv = 2", "n_kv = 4"))
    assert e.value.line == -1 and "DivisibilityViolation" in e.value.message


def test_round_trip_bit_exact(api):
    c = api.parse_config(TOY)
    c.hardware.link_bw = 8.000000001e9
    c.model.kv_dtype_bytes = 0.5
    c.policy.weights_on_gpu = 0.05
    r = api.parse_config(api.serialize_config(c))
    for part in ("hardware", "model", "workload", "policy"):
        a, b = getattr(c, part), getattr(r, part)
        assert all(getattr(a, n) == getattr(b, n) for n, _ in a._fields_)


def test_duplicate_key_line(api):
    with pytest.raises(capi.ConfigError) as e:
        api.parse_config("[hardware]\nm_g = 1\nm_g = 2\n")
    assert e.value.line == 3 and "first set on line 2" in e.value.message


def test_missing_file(api):
    with pytest.raises(capi.ConfigError) as e:
        api.parse_config_file("/nonexistent/x.cfg")
    assert e.value.line == 0 and "cannot open config file" in e.value.message


@pytest.mark.parametrize("text", [TOY, B200])
def test_known_configs_match_reference(api, ref, text):
    assert outcome(api, text) == outcome(ref, text)
    assert outcome(api, text)[0] == "ok"


VALUES = ["1.5G", "1.5g", "2TFLOPS", "2tflops", "3GFLOPS", "3e9", "1e", "", "0x10", "inf", "nan", "-1",
          "1.5", "2", " 7 ", "1 G", "G", "TFLOPS", "0", "1", "1e300", "4e-3", ".5", "5.", "+3", "1,5",
          "12K", "12k", "7T", "9M", "1.0000000000000002"]
KEYS = ["m_g", "b_cg", "p_c", "h1", "n_kv", "k", "dt_w", "s", "N", "mu", "A_g", "F_g", "r_w", "r_c", "zz"]


def mutate(rng, text):
    lines = text.splitlines()
    for _ in range(rng.randint(1, 3)):
        op = rng.randrange(9)
        i = rng.randrange(len(lines))
        if op == 0:
            del lines[i]
        elif op == 1:
            lines.insert(i, lines[rng.randrange(len(lines))])
        elif op == 2 and "=" in lines[i]:
            k = lines[i].split("=")[0]
            lines[i] = f"{k}= {rng.choice(VALUES)}"
        elif op == 3:
            lines.insert(i, f"{rng.choice(KEYS)} = {rng.choice(VALUES)}")
        elif op == 4:
            lines.insert(i, rng.choice(["[policy]", "[hardware", "[ model ]", "[bogus]", "[]", "junk",
                                        "  # only a comment", "= 3", "m_g 5"]))
        elif op == 5:
            j = rng.randrange(len(lines))
            lines[i], lines[j] = lines[j], lines[i]
        elif op == 6:
            lines = [ln for ln in lines if not ln.startswith("[policy]")]
        elif op == 7:
            lines.insert(0, f"{rng.choice(KEYS)} = 1")
        else:
            lines[i] = lines[i] + rng.choice(["  # trailing", "\t", " \r", "#", "# = 9"])
    return "\n".join(lines) + rng.choice(["\n", "", "\n\n"])


def test_mutation_fuzz_matches_reference(api, ref):
    rng = random.Random(20241117)
    kinds = {"ok": 0, "error": 0}
    for _ in range(1500):
        text = mutate(rng, rng.choice([TOY, B200]))
        a, b = outcome(api, text), outcome(ref, text)
        assert a == b, text
        kinds[a[0]] += 1
    assert kinds["ok"] > 50 and kinds["error"] > 500  # both branches exercised
