"""bench.py's bound arithmetic on CPU: the HRM bound it prints is the
reference's own estimate_throughput (planner.cpp:129-162) on the measured
spec, with the documented B200 additions — per-GPU links under TP, the
codec's stored bytes per weight, the NVLink roof.  Pinned against the
numbers BASELINE.md derives from the compiled reference (link 55 GB/s
placeholder there, 55.6 measured here)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_11217_b200 import capi  # noqa: E402

PK = {"hbm_gbs": 6548.5, "bf16_tflops": 1393.0, "bf16_tflops_sustained": 1393.0}


def _cfg(name, tp=None, codec=False):
    cfg = dict(bench.CONFIGS[name])
    if isinstance(cfg["r_w"], dict):
        cfg["r_w"] = cfg["r_w"][tp]
    cfg["codec"] = codec
    return cfg


def test_headline_bound_matches_baseline_md():
    # 8x7B @16 GB, r_w 0.10 -> 168.4 tok/s at b_cg = 55 GB/s (link bound)
    b = bench.hrm_bound(_cfg("mixtral8x7b-16g"), 55.0, 300.0, PK)
    assert b.decode_throughput == pytest.approx(168.4, rel=2e-3)
    assert b.breakdown.layer_total == pytest.approx(b.breakdown.link_upload)


@pytest.mark.parametrize("name,tp,expect", [("mixtral8x22b-tp", 2, 106), ("mixtral8x22b-tp", 4, 236),
                                            ("mixtral8x22b-tp", 8, 669)])
def test_tp_bounds_match_baseline_md(name, tp, expect):
    # BASELINE.md §2 (link = tp * b_cg, b_cg = 55 GB/s, host 300 GB/s)
    b = bench.hrm_bound(_cfg(name, tp), 55.0, 300.0, PK, tp=tp, per_slice_host=True)
    assert b.decode_throughput == pytest.approx(expect, rel=0.012)


def test_codec_bound_uses_stored_bytes():
    raw = bench.hrm_bound(_cfg("mixtral8x7b-16g"), 55.6, 125.0, PK)
    cfg = _cfg("mixtral8x7b-16g", codec=True)
    assert bench.model_spec(cfg, stored=True).weight_dtype_bytes == pytest.approx(bench.CODEC_DT)
    assert bench.CODEC_DT == pytest.approx(11600 / 8192)  # the default 3-bit code (codec 4)
    assert bench.model_spec(cfg).weight_dtype_bytes == 2.0  # the runtime always computes in bf16
    same_rw = bench.hrm_bound(cfg, 55.6, 125.0, PK)
    # same residency, 29.2 % fewer streamed bytes: link-bound layer time shrinks by the byte ratio
    assert same_rw.breakdown.link_upload == pytest.approx(raw.breakdown.link_upload * bench.CODEC_DT / 2, rel=2e-3)
    cfg["r_w"] = bench.search_rw(cfg, 55.6, 125.0, PK)
    assert cfg["r_w"] > 0.10  # the same budget holds more encoded weights
    assert bench.hrm_bound(cfg, 55.6, 125.0, PK).decode_throughput > 1.35 * raw.decode_throughput


def test_bound_uses_the_runtimes_stored_bytes():
    """After runtime creation bench.py sets cfg['stored_dt'] to the runtime's
    reported bytes per weight (raw-fallback blocks, or the 12-bit code when the
    11-bit one does not fit, stream more): the executed run's bound and the
    roofline's algorithmic bytes follow it; a larger stored size lowers the
    link-bound bound by the byte ratio."""
    cfg = _cfg("mixtral8x7b-16g", codec=True)
    cfg["r_w"] = 0.18
    b0 = bench.hrm_bound(cfg, 55.6, 125.0, PK)
    cfg2 = dict(cfg, stored_dt=12432 / 8192)
    assert bench.model_spec(cfg2, stored=True).weight_dtype_bytes == pytest.approx(12432 / 8192)
    with pytest.raises(capi.InfeasiblePolicyError):   # r_w 0.18 does not fit 16 GB at 12432 B / tile
        bench.hrm_bound(cfg2, 55.6, 125.0, PK)
    cfg["r_w"] = cfg2["r_w"] = 0.15
    b0 = bench.hrm_bound(cfg, 55.6, 125.0, PK)
    b1 = bench.hrm_bound(cfg2, 55.6, 125.0, PK)
    assert b1.breakdown.link_upload == pytest.approx(b0.breakdown.link_upload * 12432 / 11600, rel=2e-3)
    assert b1.decode_throughput < b0.decode_throughput


def test_nvlink_roof_only_adds_to_gpu_term():
    cfg = _cfg("dbrx-tp", 4)
    b = bench.hrm_bound(cfg, 55.6, 125.0, PK, tp=4, per_slice_host=True)
    assert b.breakdown.layer_total == pytest.approx(b.breakdown.link_upload)  # still link bound
    assert b.breakdown.gpu_ffn > 0


def test_arena_extra_counts_embedding_and_lm_head():
    cfg = _cfg("mixtral8x7b-16g")
    assert bench.arena_extra(cfg) == pytest.approx(2 * 32000 * 4096 * 2 + 0.2e9)
