"""Oracle: load balancer, per-node Priority Buffers and the multi-worker scheduling simulator.
TEST INFRASTRUCTURE ONLY (imported by tests/, bench.py's cpu_baseline / reference arm).

SURVEY.md Sec. 8f rows f2 (per-node buffers + least-loaded balancer) and f3 (starvation control).

PAPER.md Algorithm 1 (alg:scheduler_flow) and Sec. 4.1:
  * "The load balancer greedily distributes the jobs among the worker processes ... selects
    the worker executing the fewest number of jobs" (Alg. 1 line 3
    `Load Balancer.get_min_load(G)`); ties -> lowest worker id;
  * "The Priority Buffer consists of multiple priority queues, where each queue stores jobs
    assigned to a specific node";
  * "Whenever a backend server becomes available, a batched prompt is formed, starting with the
    prompt with the highest priority": each node's batch comes from its own queue only.
Event order at one instant t (reading R18): (a) windows ending at t complete (their
finished jobs leave the node's load), (b) jobs arriving at or before t are admitted in arrival
order, each to the then least-loaded node, (c) every free worker, in id order, forms a batch.
With one worker this is exactly oracle.sim.simulate.
"""
from __future__ import annotations

import numpy as np

from .select import isrtf_select, POLICY_ISRTF, POLICY_FCFS  # noqa: F401  (re-exported)
from .sim import oracle_remaining


def assign_nodes(load, n_new: int):
    """Greedy least-loaded assignment of n_new jobs arriving in order (Alg. 1 line 3).

    Returns (node ids int32 [n_new], updated load int64 [W]).  Each job goes to the node with
    the fewest assigned jobs at its arrival, ties to the lowest node id, and raises that load."""
    load = np.array(load, dtype=np.int64).copy()
    if load.size == 0:
        raise ValueError("no worker nodes")
    out = np.empty(n_new, dtype=np.int32)
    for j in range(n_new):
        w = int(np.argmin(load))          # first minimum = lowest id among ties
        out[j] = w
        load[w] += 1
    return out, load


def select_nodes(pred, generated, node, num_nodes: int, batch_cap: int, policy: int = POLICY_ISRTF,
                 allow_preempt: bool = True, order=None, running=None, node_ready=None,
                 head_predicts_total: bool = False, windows_waited=None, boost_after: int = 1,
                 boost_amount: float = 0.0, preempt_margin: float = 0.0):
    """Per-node Batcher.batch: for every ready node w, the batch_cap highest-priority eligible
    slots among those with node[i] == w.

    Returns (out_ids int32 [num_nodes, batch_cap] -1 padded, counts int32 [num_nodes],
    preempted uint8 [n], nan_count).  A slot of a node that is not ready is never selected nor
    flagged.  Per node this is isrtf_select on that node's slots."""
    pred = np.asarray(pred, dtype=np.float32)
    n = pred.shape[0]
    generated = np.asarray(generated, dtype=np.int64)
    node = np.asarray(node, dtype=np.int64)
    order = np.arange(n, dtype=np.uint64) if order is None else np.asarray(order, dtype=np.uint64)
    running = np.zeros(n, dtype=np.uint8) if running is None else np.asarray(running, dtype=np.uint8)
    ready = np.ones(num_nodes, dtype=bool) if node_ready is None else np.asarray(node_ready, dtype=bool)
    waited = None if windows_waited is None else np.asarray(windows_waited, dtype=np.int64)
    out_ids = np.full((num_nodes, max(batch_cap, 0)), -1, dtype=np.int32)
    counts = np.zeros(num_nodes, dtype=np.int32)
    preempted = np.zeros(n, dtype=np.uint8)
    nan_total = 0
    for w in range(num_nodes):
        idx = np.nonzero(node == w)[0]
        if not ready[w]:
            continue
        ids, cnt, pre, nan = isrtf_select(pred[idx], generated[idx], batch_cap, policy, allow_preempt,
                                          order[idx], running[idx], head_predicts_total,
                                          None if waited is None else waited[idx], boost_after,
                                          boost_amount, preempt_margin)
        out_ids[w, :cnt] = idx[ids[:cnt]]
        counts[w] = cnt
        preempted[idx] = pre
        nan_total += nan
    return out_ids, counts, preempted, nan_total


def simulate_nodes(jobs, workers: int = 1, policy: int = POLICY_ISRTF, cap: int = 1, K: int = 50,
                   ttft: float = 0.0, tpot: float = 1.0, allow_preempt: bool = True,
                   priority=oracle_remaining, boost_after: int = 1, boost_amount: float = 0.0,
                   preempt_margin: float = 0.0, trace: list | None = None):
    """Multi-worker Algorithm 1 with per-node Priority Buffers; returns {job id: (first, finish, node)}.

    Windows as in oracle.sim.simulate: min(K, smallest remaining in the batch) tokens, lasting
    TTFT (if a member runs for the first time) + TPOT x tokens.  windows_waited (aging input) of
    a job = batches its node formed without it since it last ran or arrived (reading R17).
    If ``trace`` is a list, every batch formation appends (t, node, batch ids, preempted ids)."""
    jobs = sorted(jobs, key=lambda j: (j.arrival, j.id))
    nj = len(jobs)
    rank = {j.id: r for r, j in enumerate(jobs)}
    gen = {j.id: 0 for j in jobs}
    node_of: dict = {}
    waited: dict = {}
    first, finish = {}, {}
    load = np.zeros(workers, dtype=np.int64)
    free_at = [None] * workers          # window end time of a busy worker, None = free
    batch_of = [[] for _ in range(workers)]
    tokens_of = [0] * workers
    running_prev = [set() for _ in range(workers)]
    nxt = 0
    t = 0.0
    while len(finish) < nj:
        ends = [free_at[w] for w in range(workers) if free_at[w] is not None]
        t_end = min(ends) if ends else np.inf
        t_arr = jobs[nxt].arrival if nxt < nj else np.inf
        t = min(t_end, t_arr)
        # (a) windows ending at t
        for w in range(workers):
            if free_at[w] is not None and free_at[w] <= t:
                running_prev[w] = set()
                for j in batch_of[w]:
                    gen[j.id] += tokens_of[w]
                    if gen[j.id] >= j.total:
                        finish[j.id] = free_at[w]
                        load[w] -= 1
                    else:
                        running_prev[w].add(j.id)
                free_at[w] = None
                batch_of[w] = []
        # (b) arrivals
        while nxt < nj and jobs[nxt].arrival <= t:
            w = int(np.argmin(load))
            node_of[jobs[nxt].id] = w
            waited[jobs[nxt].id] = 0
            load[w] += 1
            nxt += 1
        # (c) free workers form batches from their own queue
        for w in range(workers):
            if free_at[w] is not None:
                continue
            avail = [j for j in jobs[:nxt] if node_of[j.id] == w and j.id not in finish]
            if not avail:
                running_prev[w] = set()
                continue
            pred = np.array([priority(j, gen[j.id]) for j in avail], dtype=np.float32)
            generated = np.array([gen[j.id] for j in avail], dtype=np.int32)
            order = np.array([rank[j.id] for j in avail], dtype=np.uint32)
            running = np.array([1 if j.id in running_prev[w] else 0 for j in avail], dtype=np.uint8)
            wt = np.array([waited[j.id] for j in avail], dtype=np.int64)
            ids, count, preempted, _ = isrtf_select(pred, generated, cap, policy, allow_preempt, order, running,
                                                    False, wt, boost_after, boost_amount, preempt_margin)
            batch = [avail[i] for i in ids[:count]]
            chosen = {j.id for j in batch}
            for j in avail:
                waited[j.id] = 0 if j.id in chosen else waited[j.id] + 1
            if trace is not None:
                trace.append((t, w, [j.id for j in batch], [avail[i].id for i in np.nonzero(preempted)[0]]))
            tok = min(K, min(j.total - gen[j.id] for j in batch))
            dur = (ttft if any(j.id not in first for j in batch) else 0.0) + tpot * tok
            for j in batch:
                first.setdefault(j.id, t)
            batch_of[w], tokens_of[w], free_at[w] = batch, tok, t + dur
    return {j.id: (first[j.id], finish[j.id], node_of[j.id]) for j in jobs}
