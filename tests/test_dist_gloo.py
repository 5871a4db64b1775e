"""Multi-process (world_size 2, gloo, CPU) checks of the multi-GPU selection algorithm.

elis_isrtf_select_dist (include/elis.h) shards the in-flight slots over ranks, takes each
rank's local top-cap candidates, all-gathers them and merges identically on every rank.
It is exact because keys are globally unique (the tie-break rank of (arrival, id) is
global) and the global top-cap is contained in the union of the local top-caps.  Here the
same decomposition runs over torch.distributed (gloo) with the ORACLE select on each rank,
and must reproduce the single-process oracle select bit for bit -- including preemption
flags computed against the global threshold.  (The GPU path itself is exercised with
NCCL in tests/test_gpu_dist.py.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_09142_b200 import inputs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _key(pred, gen, order, running, allow):
    """(class, fp32 key, order) of one slot -- the oracle's sort key, for thresholds."""
    import math
    r = np.float32(pred)
    k = math.inf if math.isnan(r) else (float(r) if r > 0 else 0.0)
    return (0 if (allow or running) else 1, k, int(order))


def _worker(rank, world, port, n, cap, seed, allow, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.select import isrtf_select
    pred = inputs.random_predictions(n, seed=seed)
    gen, order, running = inputs.random_sched_state(n, seed=seed)
    shard = np.array_split(np.arange(n), world)[rank]
    lo = int(shard[0])
    # local top-cap on this rank's slots (global order ranks), ids made global
    ids, cnt, _, _ = isrtf_select(pred[shard], gen[shard], cap, 0, allow, order[shard], running[shard])
    cand = np.full(cap, -1, np.int64)
    cand[:cnt] = ids[:cnt] + lo
    t = torch.from_numpy(cand)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    allc = torch.cat(gathered).numpy()
    allc = allc[allc >= 0]
    # identical merge on every rank: oracle select over the candidates
    m_ids, m_cnt, _, _ = isrtf_select(pred[allc], gen[allc], cap, 0, allow, order[allc], running[allc])
    merged = np.full(cap, -1, np.int64)
    merged[:m_cnt] = allc[m_ids[:m_cnt]]
    # local preemption flags against the global threshold key
    thr = max(_key(pred[i], gen[i], order[i], running[i], allow) for i in merged[:m_cnt]) if m_cnt else None
    pre = np.array([int(running[i] == 1 and not (gen[i] >= 0 and thr is not None and
                                                 _key(pred[i], gen[i], order[i], running[i], allow) <= thr))
                    for i in shard], np.uint8)
    out_q.put((rank, merged.tolist(), int(m_cnt), lo, pre.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,cap,seed,allow", [(1000, 16, 1, True), (4097, 256, 2, False), (50, 64, 3, True),
                                              (65536 // 16, 4, 4, True)])
def test_distributed_topk_merge_equals_global_select(n, cap, seed, allow):
    from oracle.select import isrtf_select
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, cap, seed, allow, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pred = inputs.random_predictions(n, seed=seed)
    gen, order, running = inputs.random_sched_state(n, seed=seed)
    g_ids, g_cnt, g_pre, _ = isrtf_select(pred, gen, cap, 0, allow, order, running)
    for rank, merged, m_cnt, lo, pre in res:
        assert m_cnt == g_cnt
        assert merged == [int(x) for x in g_ids]          # identical batch on every rank
        assert pre == [int(x) for x in g_pre[lo:lo + len(pre)]]


def test_bench_reference_arm_runs_on_cpu(tmp_path):
    """bench.py --impl reference (the oracle on host cores) prints one JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--config", "tiny",
                        "--n", "16", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    for k in ("cpu_baseline", "e2e", "metric", "unit", "config"):
        assert k in line


def _shard_worker(rank, world, port, win, out_q):
    """One rank of bench.py's cfg5 multi-GPU iteration, host side: the due window is split at the
    quantiles of its encoder cost by the LIBRARY (elis_cost_split, a host function of the C ABI),
    each rank writes predictions for its slice only, the (slot, prediction) pairs are all-gathered
    into every rank's copy of the 65,536-slot table, and every rank selects over the whole table."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle.select import isrtf_select
    cfg = inputs.CONFIGS["base"]
    F, due = 65536, -(-65536 // inputs.WINDOW_K)
    Lt = np.asarray(inputs.trace_lengths(F, seed=0)[0], np.int32)
    slots = bench.due_windows(F, due)[win]
    b = bench.cost_bounds(Lt[slots], world, cfg)
    mine = slots[b[rank]:b[rank + 1]]
    # stand-in for this rank's encoder output: any deterministic function of the slot
    pred_all = inputs.random_predictions(F, seed=win)
    table = np.zeros(F, np.float32)
    pairs = np.full((due, 2), -1.0, np.float64)
    pairs[:len(mine), 0] = mine
    pairs[:len(mine), 1] = pred_all[mine]
    t = torch.from_numpy(pairs)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    for g in gathered:
        g = g.numpy()
        g = g[g[:, 0] >= 0]
        table[g[:, 0].astype(np.int64)] = g[:, 1].astype(np.float32)
    gen, order, running = inputs.random_sched_state(F, seed=win)
    ids, cnt, _, _ = isrtf_select(table, gen, 256, 0, True, order, running)
    out_q.put((rank, [int(x) for x in b], mine.tolist(), ids[:cnt].tolist(), table[slots].tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,win", [(2, 0), (4, 7)])
def test_cfg5_due_set_sharding_over_ranks(world, win):
    """bench.py's cfg5 sharding over `world` gloo ranks: every rank computes the same cost bounds
    (library call), the slices partition the due window, each rank's encoder cost is within one
    request of the ideal share, and the gathered table -- hence the ISRTF batch -- is the
    single-process one on every rank."""
    import bench
    from oracle.select import isrtf_select
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, win, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    F, due = 65536, -(-65536 // inputs.WINDOW_K)
    Lt = np.asarray(inputs.trace_lengths(F, seed=0)[0], np.int32)
    slots = bench.due_windows(F, due)[win]
    bounds = [r[1] for r in res]
    assert all(bb == bounds[0] for bb in bounds)
    assert sorted(s for r in res for s in r[2]) == sorted(slots.tolist())  # a partition of the window
    L = Lt[slots].astype(np.float64)
    cost = 169.87e6 * L + 36864.0 * L * L
    share = [cost[bounds[0][r]:bounds[0][r + 1]].sum() for r in range(world)]
    assert max(share) - cost.sum() / world <= cost.max()
    pred_all = inputs.random_predictions(F, seed=win)
    table = np.zeros(F, np.float32)
    table[slots] = pred_all[slots]
    gen, order, running = inputs.random_sched_state(F, seed=win)
    ids, cnt, _, _ = isrtf_select(table, gen, 256, 0, True, order, running)
    for r in res:
        assert r[3] == ids[:cnt].tolist()
        np.testing.assert_array_equal(np.asarray(r[4], np.float32), table[slots])  # NaN slots included
