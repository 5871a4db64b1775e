"""Host-side logic of bench.py (no GPU): argument parsing (the torchrun-safe --requests alias),
the L2 policy that decides when a timed step must be preceded by an L2 flush, and the JSON
config description."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(*argv):
    old = sys.argv
    sys.argv = ["bench.py", *argv]
    try:
        a = bench.parse()
    finally:
        sys.argv = old
    a.residual = a.residual or "fp32"
    a.transport_used = "none"
    return a


def test_requests_alias_and_defaults():
    a = _args("--requests", "64")
    assert a.n == 64 and a.gpus == 1 and a.graph == "on" and a.transport == "peer"
    assert _args("--n", "32").n == 32


def test_l2_policy_flushes_only_small_working_sets():
    tiny = _args("--config", "tiny")
    flush, why = bench.l2_policy(tiny, 16 * 64)
    assert flush and "flushed" in why
    base = _args("--config", "base")
    flush, why = bench.l2_policy(base, 43296)
    assert not flush and "exceeds" in why
    # the working set grows with the tokens and with the fp32 residual stream
    assert bench.working_set_bytes(base, 2000) < bench.working_set_bytes(base, 4000)
    r16 = _args("--config", "base", "--residual", "fp16")
    assert bench.working_set_bytes(r16, 4000) < bench.working_set_bytes(base, 4000)


def test_config_description_names_the_workload():
    a = _args()
    a.precision = "fp16"
    d = bench.config_desc(a, 43296, 1)
    assert d["workload"].startswith("cfg2") and d["requests_per_gpu"] == 256 and "l2" in d
    a.transport_used = "peer (NVLink stores + epoch flags, fused select kernel)"
    d8 = bench.config_desc(a, 43296, 8)
    assert d8["transport"].startswith("peer") and "dp8" in d8["parallelism"]


def test_strong_scaling_slices_one_population():
    """--total-requests: every N sees the same request population; rank r's slice is contiguous."""
    import numpy as np
    a = _args("--total-requests", "64", "--config", "tiny")
    a.n = 64
    L, _, tok = bench.workload(a, 0)
    a.n = 16
    parts = [bench.workload(a, r) for r in range(4)]
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), L)
    np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), tok)
