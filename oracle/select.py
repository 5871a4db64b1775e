"""Oracle: ISRTF / FCFS batch selection with preemption flags.  TEST INFRASTRUCTURE ONLY.

PAPER.md Algorithm 1 (alg:scheduler_flow) lines 10-19: every job
returned to the Job Pool gets a priority (Predictor.init / .iter) and is pushed
to the Priority Buffer; "a batched prompt is formed, starting with the prompt
with the highest priority".  ISRTF priority = predicted remaining
tokens, smallest first; FCFS priority = arrival time.
Preemption: "vLLM will check the priority of each task and preempt the tasks
starting with the lowest priority".

DESIGN.md readings used here: R4 (head output = remaining; optional
``head_predicts_total`` subtracts generated), R5 (negative -> 0,
-0 -> +0, NaN -> +inf, counted), R6 (ties -> arrival rank, then id: ``order``
is the unique rank of (arrival, id)), R9 (allow_preempt semantics), R10 (batch
order ascending), R11 (underfull batch, -1 padding).

The decision "which key is smaller" is taken in fp32, the precision the GPU
path keys in, so both sides order identical fp32 values identically.
"""
from __future__ import annotations

import math

import numpy as np

POLICY_ISRTF = 0
POLICY_FCFS = 1


def starvation_adjust(rem: float, waited: int, is_running: bool, boost_after: int, boost_amount: float,
                      preempt_margin: float) -> float:
    """Starvation control ("policies that can adjust
    the frequency of preemption and prevent starvation"; reading R17):
      aging: subtract boost_amount x floor(windows_waited / boost_after) from the
        key (the max(0, .) floor is applied by the caller);
      preemption margin: a running job's key is lowered by preempt_margin tokens, so a waiting
        job displaces it only when predicted shorter by more than the margin.
    fp32 arithmetic, one rounding per step (the precision the keys are compared in)."""
    r = np.float32(rem)
    if boost_amount != 0.0 and waited > 0:
        r = np.float32(r - np.float32(np.float32(boost_amount) * np.float32(waited // boost_after)))
    if is_running and preempt_margin != 0.0:
        r = np.float32(r - np.float32(preempt_margin))
    return float(r)


def isrtf_select(pred, generated, batch_cap: int, policy: int = POLICY_ISRTF,
                 allow_preempt: bool = True, order=None, running=None,
                 head_predicts_total: bool = False, windows_waited=None, boost_after: int = 1,
                 boost_amount: float = 0.0, preempt_margin: float = 0.0):
    """Return (out_ids int32 [batch_cap] padded with -1, out_count, preempted uint8 [n], nan_count).

    Sorted by (class, key, order) over eligible slots (generated >= 0), where
    class = 0 for every slot when allow_preempt, else 0 for running slots and 1
    for the rest (running jobs keep their slots); key = remaining tokens (ISRTF)
    or 0 (FCFS: arrival rank alone decides).  Optional starvation control
    (ISRTF only): see starvation_adjust."""
    pred = np.asarray(pred, dtype=np.float32)
    generated = np.asarray(generated, dtype=np.int64)
    n = pred.shape[0]
    order = np.arange(n, dtype=np.uint64) if order is None else np.asarray(order, dtype=np.uint64)
    running = np.zeros(n, dtype=np.uint8) if running is None else np.asarray(running, dtype=np.uint8)
    waited = None if windows_waited is None else np.asarray(windows_waited, dtype=np.int64)
    if boost_after < 1:
        raise ValueError("boost_after must be >= 1")
    nan_count = 0
    items = []
    for i in range(n):
        if generated[i] < 0:
            continue
        if policy == POLICY_ISRTF:
            p = np.float32(pred[i])
            rem = np.float32(p - np.float32(generated[i])) if head_predicts_total else p
            if math.isnan(float(rem)):
                nan_count += 1
                k = math.inf
            else:
                adj = starvation_adjust(float(rem), int(waited[i]) if waited is not None else 0,
                                        bool(running[i]), boost_after, boost_amount, preempt_margin)
                k = adj if adj > 0.0 else 0.0
        elif policy == POLICY_FCFS:
            k = 0.0
        else:
            raise ValueError("unknown policy")
        cls = 0 if (allow_preempt or running[i]) else 1
        items.append(((cls, k, int(order[i])), i))
    items.sort(key=lambda t: t[0])
    take = min(max(batch_cap, 0), len(items))
    chosen = [i for _, i in items[:take]]
    out_ids = np.full(max(batch_cap, 0), -1, dtype=np.int32)
    out_ids[:take] = chosen
    selected = np.zeros(n, dtype=bool)
    selected[chosen] = True
    preempted = ((running != 0) & ~selected).astype(np.uint8)
    return out_ids, take, preempted, nan_count
