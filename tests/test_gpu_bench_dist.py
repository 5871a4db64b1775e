"""bench.py's N > 1 path on one B200: torchrun with 2 ranks sharing cuda:0 (ELIS_BENCH_SHARE_GPU=1,
gloo control plane) runs the same code as the driver's multi-GPU bench -- peer-memory transport
attached through CUDA IPC, graph capture of predict + elis_isrtf_select_dist, barriers, max over
ranks, one JSON line from rank 0.  Timings are meaningless here (the ranks share one GPU); the test
checks that the path completes and reports what ran."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra", [["--workload", "cfg1"], ["--workload", "cfg5", "--config", "tiny", "--inflight", "4096",
                                                          "--due", "96"],
                                   ["--workload", "cfg5", "--config", "tiny", "--inflight", "4096", "--due", "96",
                                    "--graph", "off"],
                                   ["--workload", "cfg1", "--graph", "off"],
                                   ["--workload", "cfg1", "--total-requests", "32"]])
def test_bench_two_ranks_peer_transport(cuda_lib, extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", *extra]
    env = {**os.environ, "ELIS_BENCH_SHARE_GPU": "1"}
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["timing"]["transport"].startswith("peer"), d["timing"]   # NCCL needs one GPU per rank
    if "--total-requests" in extra:
        assert d["scaling"] == "strong" and d["config"]["requests_per_gpu"] == 16
    if "cfg5" in extra:
        assert d["scaling"] == "strong" and d["config"]["due_per_iteration"] == 96
        assert sum(d["sharding"]["rank_requests_window0"]) == 96
    if "--graph" not in extra:
        assert d["timing"]["cuda_graph"].startswith("on"), d["timing"]
