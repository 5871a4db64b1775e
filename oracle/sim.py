"""Oracle: window-level scheduling simulator for the JCT pins.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md Algorithm 1 (alg:scheduler_flow) and Sec. 4.1
 for one backend worker:
  * every scheduling iteration re-prioritises the jobs (lines 10-18) and forms a
    batch "starting with the prompt with the highest priority" (line 19);
  * the batch executes one window of K = 50 tokens -- the
    backend returns "when all prompts in the batch have produced K tokens or
    when a prompt has finished", so a window lasts min(K, min remaining
    over the batch) tokens (reading R15);
  * unfinished jobs go back to the pool (lines 24-26).
Window duration = TTFT (if a member runs for the first time) + TPOT x tokens
(Sec. 2.1 latency model).  Arrivals are seen at the next
window boundary; an idle worker jumps to the next arrival.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .select import isrtf_select, POLICY_ISRTF, POLICY_FCFS


@dataclass
class SimJob:
    id: int
    arrival: float       # ms
    total: int           # true output tokens (>= 1)


def oracle_remaining(job: SimJob, generated: int) -> float:
    """Perfect predictor: remaining = total - generated (Fig. 2(a): 120 -> 70)."""
    return float(job.total - generated)


def simulate(jobs, policy: int = POLICY_ISRTF, cap: int = 1, K: int = 50, ttft: float = 0.0,
             tpot: float = 1.0, allow_preempt: bool = True, priority=oracle_remaining,
             trace: list | None = None):
    """Run to completion; returns {job id: (first_exec, finish)}.

    ``priority(job, generated)`` gives the ISRTF key (predicted remaining);
    ignored for FCFS.  If ``trace`` is a list, each iteration appends
    (t, batch ids, preempted ids)."""
    jobs = sorted(jobs, key=lambda j: (j.arrival, j.id))
    rank = {j.id: r for r, j in enumerate(jobs)}          # order = rank of (arrival, id)
    gen = {j.id: 0 for j in jobs}
    first, finish = {}, {}
    running_prev: set = set()
    t = 0.0
    while len(finish) < len(jobs):
        avail = [j for j in jobs if j.arrival <= t and j.id not in finish]
        if not avail:
            t = min(j.arrival for j in jobs if j.id not in finish)
            running_prev = set()
            continue
        pred = np.array([priority(j, gen[j.id]) for j in avail], dtype=np.float32)
        generated = np.array([gen[j.id] for j in avail], dtype=np.int32)
        order = np.array([rank[j.id] for j in avail], dtype=np.uint32)
        running = np.array([1 if j.id in running_prev else 0 for j in avail], dtype=np.uint8)
        ids, count, preempted, _ = isrtf_select(pred, generated, cap, policy, allow_preempt,
                                                order, running)
        batch = [avail[i] for i in ids[:count]]
        if trace is not None:
            trace.append((t, [j.id for j in batch],
                          [avail[i].id for i in np.nonzero(preempted)[0]]))
        w = min(K, min(j.total - gen[j.id] for j in batch))
        dur = (ttft if any(j.id not in first for j in batch) else 0.0) + tpot * w
        for j in batch:
            first.setdefault(j.id, t)
        t += dur
        running_prev = set()
        for j in batch:
            gen[j.id] += w
            if gen[j.id] >= j.total:
                finish[j.id] = t
            else:
                running_prev.add(j.id)
    return {j.id: (first[j.id], finish[j.id]) for j in jobs}


def mean_jct(jobs, result) -> float:
    return float(np.mean([result[j.id][1] - j.arrival for j in jobs]))


def static_priority(order_of_ids):
    """Priority function for a fixed (static) job order: rank in ``order_of_ids``."""
    pos = {jid: r for r, jid in enumerate(order_of_ids)}
    return lambda job, generated: float(pos[job.id])
