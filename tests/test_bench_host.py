"""Host-side logic of bench.py (no GPU): argument parsing (workload presets, the torchrun-safe
--requests alias), the cfg5 due windows (every in-flight slot re-predicted), the L2
policy that decides when a timed step must be preceded by an L2 flush, the JSON config
description shared by both arms, and the roofline arithmetic."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2505_09142_b200 import inputs  # noqa: E402


def _args(*argv):
    a = bench.parse(list(argv))
    a.residual = a.residual or "fp32"
    return a


def test_default_is_the_north_star_workload():
    a = bench.parse([])
    assert a.workload == "cfg5" and a.config == "base" and a.inflight == 65536
    assert a.due == 1311 == -(-65536 // 50) and a.cap == 256 and a.gpus == 1
    assert a.graph == "on" and a.transport == "peer"


def test_workload_presets_and_requests_alias():
    a = _args("--workload", "cfg2")
    assert a.inflight == 0 and a.n == 256 and a.cap == 4 and a.config == "base"
    assert _args("--workload", "cfg2", "--requests", "64").n == 64
    assert _args("--workload", "cfg2", "--n", "32").n == 32
    t = _args("--workload", "cfg1")
    assert t.config == "tiny" and t.n == 16 and t.lengths == "fixed:64"
    legacy = _args("--config", "tiny", "--requests", "16", "--inflight", "4096", "--gpus", "2")
    assert legacy.inflight == 4096 and legacy.due == 32


def test_due_windows_cover_every_slot():
    for F, due in ((65536, 1311), (4096, 64), (1000, 333)):
        wins = bench.due_windows(F, due)
        assert all(len(w) == due for w in wins)
        assert len(wins) == -(-F // due)
        assert np.array_equal(np.unique(np.concatenate(wins)), np.arange(F))


def test_l2_policy_flushes_only_small_working_sets():
    tiny = _args("--workload", "cfg1")
    flush, why = bench.l2_policy(tiny, 16 * 64)
    assert flush and "flushed" in why
    base = _args("--workload", "cfg2")
    flush, why = bench.l2_policy(base, 43296)
    assert not flush and "exceeds" in why
    # the working set grows with the tokens and with the fp32 residual stream
    assert bench.working_set_bytes(base, 2000) < bench.working_set_bytes(base, 4000)
    r16 = _args("--workload", "cfg2", "--residual", "fp16")
    assert bench.working_set_bytes(r16, 4000) < bench.working_set_bytes(base, 4000)


def test_config_description_names_the_workload_and_is_arm_independent():
    a = _args("--workload", "cfg2")
    d = bench.config_desc(a, 43296, 1)
    assert d["workload"].startswith("cfg2") and d["requests_per_gpu"] == 256 and "l2" in d
    d8 = bench.config_desc(a, 8 * 43296, 8)
    assert "dp8" in d8["parallelism"] and d8["tokens_per_gpu_step"] == 43296
    c5 = bench.config_desc(_args(), 222000, 8)
    assert c5["workload"].startswith("cfg5") and c5["due_per_iteration"] == 1311 and c5["inflight"] == 65536
    # nothing arm- or run-specific (graph mode, transport, precision) inside config
    for k in ("cuda_graph", "transport", "precision", "residual"):
        assert k not in c5 and k not in d


def test_strong_scaling_slices_one_population():
    """--total-requests: every N sees the same request population; rank r's slice is contiguous."""
    a = _args("--workload", "cfg1", "--total-requests", "64")
    a.n = 64
    L, _, tok = bench.workload(a, 0)
    a.n = 16
    parts = [bench.workload(a, r) for r in range(4)]
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), L)
    np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), tok)


def test_roofline_arithmetic():
    """The roofline object recomputes by hand: achieved = algorithmic FLOPs per launch / launch
    time; the burst peak below 4 s of timed region; the whole-step fraction = sum of ideal times."""
    cfg = inputs.CONFIGS["base"]
    T, n, sL2 = 10000.0, 60.0, 60 * 170.0 ** 2
    work = bench.step_work(cfg, T, n, sL2, 65536, True)
    peaks = {"bf16_tflops": 1678.0, "bf16_tflops_sustained": 1410.7, "hbm_gbs": 6528.7, "sm_max_mhz": 1965.0}
    pk = bench.peaks_for(peaks, 0.5)
    assert pk["tensor_kind"] == "burst" and pk["tensor_tflops"] == 1678.0
    assert bench.peaks_for(peaks, 5.0)["tensor_kind"] == "sustained"
    steps = 4
    ffn1_us = 500.0
    prof = {"gemm_ffn1": (steps * 12 * ffn1_us / 1e3, steps * 12), "attention": (steps * 12 * 0.1, steps * 12)}
    r = bench.roofline_report(prof, steps, work, pk, 10.0, {"cfg5/fp16-r16/gemm_ffn1": 123}, "cfg5/fp16-r16")
    fl = 2.0 * T * 768 * 3072
    assert r["kernel"] == "gemm_ffn1" and r["bound"] == "tensor"
    assert abs(r["achieved"] - fl / (ffn1_us * 1e-6) / 1e12) < 0.01
    assert abs(r["frac"] - r["achieved"] / 1678.0) < 1e-3 and r["traffic"] == 123
    ideal = 12 * fl / 1678e12 * 1e3 + bench.ideal_ms(work["attention"], pk) * 12
    assert abs(r["step_ideal_ms"] - ideal) < 1e-3 and abs(r["step_frac"] - ideal / 10.0) < 1e-3
    assert set(r["attention"]) >= {"tensor_frac", "hbm_frac", "mufu_frac"}
