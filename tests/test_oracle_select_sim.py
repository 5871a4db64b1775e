"""Pins for oracle/select.py and oracle/sim.py.

  * SPEC.md worked vectors and the paper's Fig. 2(a)
    numbers (120 -> 70);
  * brute force over all subsets on tiny inputs: exactly one subset has every
    member ordered before every non-member; the oracle must return it;
  * hand-derived JCT examples from the scheduling definition (Alg. 1, P:244-272;
    window end rule P:342) -- SURVEY.md Sec. 8c "Worked JCT example";
  * brute force over all n! static priority orders: SRTF (ISRTF with a perfect
    predictor) attains the minimum mean JCT on a single server (BASELINE.json).
"""
import itertools
import math

import numpy as np
import pytest

from paper_2505_09142_b200 import inputs
from oracle.select import isrtf_select, POLICY_ISRTF, POLICY_FCFS
from oracle import sim


# ---------------------------------------------------------------- SPEC / paper vectors

def test_spec_isrtf_order():
    """ISRTF, remaining [30, 200, 10] -> buffer order [10, 30, 200]."""
    ids, cnt, _, _ = isrtf_select(np.float32([30, 200, 10]), [0, 0, 0], 3)
    assert list(ids) == [2, 0, 1] and cnt == 3


def test_spec_fcfs_order():
    """FCFS, arrivals [5 s, 1 s, 3 s] -> order [1, 3, 5]."""
    arrivals = [5.0, 1.0, 3.0]
    order = np.argsort(np.argsort(arrivals)).astype(np.uint32)   # rank of arrival
    ids, cnt, _, _ = isrtf_select(np.float32([7, 8, 9]), [0, 0, 0], 3, POLICY_FCFS, order=order)
    assert [arrivals[i] for i in ids] == [1.0, 3.0, 5.0]


def test_spec_form_batch_prefix_and_underfull():
    """buffer [10, 30, 200, 400], cap 2 -> [10, 30]; 1 job, cap 4 -> batch of 1."""
    ids, cnt, _, _ = isrtf_select(np.float32([200, 10, 400, 30]), [0] * 4, 2)
    assert list(ids) == [1, 3] and cnt == 2
    ids, cnt, _, _ = isrtf_select(np.float32([5]), [0], 4)
    assert list(ids) == [0, -1, -1, -1] and cnt == 1


def test_empty_buffer_is_noop():
    """S:275 EmptyBuffer -> no-op: count 0, all -1."""
    ids, cnt, pre, _ = isrtf_select(np.float32([]), np.zeros(0, np.int32), 3)
    assert cnt == 0 and list(ids) == [-1, -1, -1] and pre.size == 0
    ids, cnt, _, _ = isrtf_select(np.float32([1, 2]), [-1, -1], 3)
    assert cnt == 0


def test_tie_break_arrival_then_id_and_preempt_suffix():
    """Ties broken by earlier arrival then id; eviction hits the later
    arrival first: preempted = running jobs outside the top-cap."""
    pred = np.float32([50, 50, 50, 10])
    order = np.uint32([2, 0, 1, 3])            # rank of (arrival, id)
    running = np.uint8([1, 1, 1, 0])
    ids, cnt, pre, _ = isrtf_select(pred, [0, 0, 0, 0], 3, order=order, running=running)
    assert list(ids) == [3, 1, 2]
    assert list(pre) == [1, 0, 0, 0]          # the latest arrival among the tied is evicted


def test_fig2a_remaining_70():
    """Fig. 2(a): total 120, after 50 generated the remaining estimate is 70."""
    job = sim.SimJob(0, 0.0, 120)
    assert sim.oracle_remaining(job, 0) == 120 and sim.oracle_remaining(job, 50) == 70
    # head_predicts_total reading: key = max(0, total - generated)
    ids, _, _, _ = isrtf_select(np.float32([120, 75]), [50, 0], 2, head_predicts_total=True)
    assert list(ids) == [0, 1]                 # 70 < 75


def test_key_canonicalisation():
    """R5: negative -> 0, -0 -> +0 (ties with 0 broken by order), NaN -> +inf (last, counted)."""
    pred = np.float32([np.nan, -5.0, -0.0, 0.0, np.inf, 3.0])
    ids, cnt, _, nan = isrtf_select(pred, [0] * 6, 6)
    assert list(ids) == [1, 2, 3, 5, 0, 4] and nan == 1


def test_no_preempt_keeps_running_jobs():
    """allow_preempt = 0: running jobs keep their slots; free slots filled in ISRTF order."""
    pred = np.float32([500, 1, 2, 3])
    running = np.uint8([1, 0, 0, 0])
    ids, _, pre, _ = isrtf_select(pred, [0] * 4, 2, allow_preempt=False, running=running)
    assert list(ids) == [0, 1] and pre.sum() == 0
    ids, _, pre, _ = isrtf_select(pred, [0] * 4, 2, allow_preempt=True, running=running)
    assert list(ids) == [1, 2] and list(pre) == [1, 0, 0, 0]


# ---------------------------------------------------------------- brute force

def _brute_force(pred, gen, cap, policy, allow_preempt, order, running, hpt):
    """Enumerate every subset of eligible slots of the required size; keep the ones in
    which every member precedes every non-member under (class, key, order)."""
    n = len(pred)
    def k(i):
        if policy == POLICY_FCFS:
            v = 0.0
        else:
            r = np.float32(np.float32(pred[i]) - np.float32(gen[i])) if hpt else np.float32(pred[i])
            v = math.inf if math.isnan(r) else (float(r) if r > 0 else 0.0)
        c = 0 if (allow_preempt or running[i]) else 1
        return (c, v, int(order[i]))
    elig = [i for i in range(n) if gen[i] >= 0]
    size = min(cap, len(elig))
    good = []
    for S in itertools.combinations(elig, size):
        rest = [j for j in elig if j not in S]
        if all(k(i) < k(j) for i in S for j in rest):
            good.append(sorted(S, key=k))
    assert len(good) == 1
    return good[0]


@pytest.mark.parametrize("seed", range(60))
def test_select_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 9))
    pred = inputs.random_predictions(n, seed=seed)
    gen, order, running = inputs.random_sched_state(n, seed=seed, frac_running=0.3, frac_empty=0.15)
    cap = int(rng.choice([1, max(1, n - 1), n, n + 3]))
    policy = int(rng.integers(0, 2))
    allow = bool(rng.integers(0, 2))
    hpt = bool(rng.integers(0, 2))
    ids, cnt, pre, _ = isrtf_select(pred, gen, cap, policy, allow, order, running, hpt)
    bf = _brute_force(pred, gen, cap, policy, allow, order, running, hpt)
    assert list(ids[:cnt]) == bf and all(x == -1 for x in ids[cnt:])
    sel = set(bf)
    assert list(pre) == [int(running[i] == 1 and i not in sel) for i in range(n)]


def test_select_invariants_large():
    """n = 4096: |batch| = min(cap, #eligible); every selected key < every unselected one."""
    n, cap = 4096, 256
    pred = inputs.random_predictions(n, seed=11)
    gen, order, running = inputs.random_sched_state(n, seed=11)
    ids, cnt, pre, _ = isrtf_select(pred, gen, cap, order=order, running=running)
    elig = gen >= 0
    assert cnt == min(cap, int(elig.sum()))
    def key(i):
        r = pred[i]
        return (math.inf if math.isnan(r) else max(float(r), 0.0), int(order[i]))
    sel = ids[:cnt]
    worst = max(key(i) for i in sel)
    assert all(key(i) > worst for i in np.nonzero(elig)[0] if i not in set(sel))
    assert [key(i) for i in sel] == sorted(key(i) for i in sel)


# ---------------------------------------------------------------- JCT worked examples

def _jobs(spec):
    return [sim.SimJob(i, float(a), int(t)) for i, (a, t) in enumerate(spec)]


def test_worked_example_fig2a_jobs_cap1():
    """A (arrives 0, 120 tokens -- the Fig. 2(a) job), B (arrives 10 ms, 30 tokens),
    cap 1, K = 50, TPOT 1 ms, TTFT 0.  FCFS: A 120, B 150 -> mean 130.
    ISRTF + preemption: at t = 50 A's remaining is 70 vs B's 30 -> B runs
    50-80, A 80-150 -> mean (150 + 70) / 2 = 110.  ISRTF without preemption: 130."""
    jobs = _jobs([(0, 120), (10, 30)])
    f = sim.simulate(jobs, POLICY_FCFS, cap=1)
    assert f[0][1] == 120 and f[1][1] == 150 and sim.mean_jct(jobs, f) == 130
    tr = []
    s = sim.simulate(jobs, POLICY_ISRTF, cap=1, trace=tr)
    assert s[1][1] == 80 and s[0][1] == 150 and sim.mean_jct(jobs, s) == 110
    assert tr[1] == (50.0, [1], [0])           # t=50 select returns [B], A flagged preempted
    n = sim.simulate(jobs, POLICY_ISRTF, cap=1, allow_preempt=False)
    assert sim.mean_jct(jobs, n) == 130


def test_worked_example_cap2():
    """cap 2: A (0, 120), B (0, 30), C (0, 75), D (5 ms, 20).
    FCFS mean 93.75 (A 120, B 30, C 105, D 120); ISRTF mean 80 (B 30, D 45, C 75, A 170)."""
    jobs = _jobs([(0, 120), (0, 30), (0, 75), (5, 20)])
    f = sim.simulate(jobs, POLICY_FCFS, cap=2)
    assert [f[i][1] - jobs[i].arrival for i in range(4)] == [120, 30, 105, 120]
    s = sim.simulate(jobs, POLICY_ISRTF, cap=2)
    assert [s[i][1] - jobs[i].arrival for i in range(4)] == [170, 30, 75, 45]
    assert sim.mean_jct(jobs, f) == 93.75 and sim.mean_jct(jobs, s) == 80


def test_spec_500_and_nine_10s():
    """[500 x 1, 10 x 9] simultaneous, cap 1: FCFS 545 vs ISRTF 104."""
    jobs = _jobs([(0, 500)] + [(0, 10)] * 9)
    assert sim.mean_jct(jobs, sim.simulate(jobs, POLICY_FCFS, cap=1)) == 545
    assert sim.mean_jct(jobs, sim.simulate(jobs, POLICY_ISRTF, cap=1)) == 104


def test_single_job_latency_formula():
    """One job, no contention: JCT = TTFT + TPOT x tokens (S:... 'run' example)."""
    jobs = _jobs([(3, 137)])
    r = sim.simulate(jobs, POLICY_ISRTF, cap=4, ttft=20.0, tpot=2.0)
    assert r[0][1] - 3 == 20.0 + 2.0 * 137


@pytest.mark.parametrize("seed", range(40))
def test_srtf_minimises_mean_jct_brute_force(seed):
    """Single server, cap 1, simultaneous arrivals, n <= 6: ISRTF with a perfect
    predictor equals the minimum mean JCT over all n! static priority orders."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 7))
    jobs = _jobs([(0, int(t)) for t in rng.integers(1, 300, n)])
    isrtf = sim.mean_jct(jobs, sim.simulate(jobs, POLICY_ISRTF, cap=1))
    best = min(sim.mean_jct(jobs, sim.simulate(jobs, POLICY_ISRTF, cap=1,
                                               priority=sim.static_priority(p)))
               for p in itertools.permutations(range(n)))
    assert isrtf == pytest.approx(best, abs=1e-9)
    assert isrtf <= sim.mean_jct(jobs, sim.simulate(jobs, POLICY_FCFS, cap=1)) + 1e-9


@pytest.mark.parametrize("seed", range(20))
def test_srtf_staggered_arrivals_cap1(seed):
    """Staggered arrivals, cap 1: ISRTF (perfect predictor, preemptive at window
    boundaries) is no worse than any static priority order."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(2, 6))
    jobs = _jobs([(int(a), int(t)) for a, t in zip(rng.integers(0, 200, n), rng.integers(1, 250, n))])
    isrtf = sim.mean_jct(jobs, sim.simulate(jobs, POLICY_ISRTF, cap=1))
    best = min(sim.mean_jct(jobs, sim.simulate(jobs, POLICY_ISRTF, cap=1,
                                               priority=sim.static_priority(p)))
               for p in itertools.permutations(range(n)))
    assert isrtf <= best + 1e-9
