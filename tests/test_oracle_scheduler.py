"""Pins for oracle/scheduler.py (load balancer, per-node Priority Buffers, multi-worker
simulator) and the starvation controls of oracle/select.py.

  * SPEC.md worked vectors for the load balancer (loads [3,1,2] -> 1, [2,2,2] -> 0,
    100 submissions on 4 idle workers -> 25 each) and for per-node batches;
  * hand-derived multi-worker JCTs from Algorithm 1 and the window rule;
  * cross-check: the multi-worker simulator with one worker equals the independently written
    single-worker simulator (oracle.sim.simulate) on random streams;
  * aging / margin closed forms and a starvation bound derived by hand.
"""
import numpy as np
import pytest

from oracle import scheduler, sim
from oracle.select import isrtf_select, POLICY_FCFS, POLICY_ISRTF


def _jobs(spec):
    return [sim.SimJob(i, float(a), int(t)) for i, (a, t) in enumerate(spec)]


# ---------------------------------------------------------------- load balancer (Alg. 1 line 3)

def test_spec_least_loaded():
    assert scheduler.assign_nodes([3, 1, 2], 1)[0].tolist() == [1]
    assert scheduler.assign_nodes([2, 2, 2], 1)[0].tolist() == [0]      # S:258 ties -> lowest id


def test_spec_uniform_stream_balances():
    nodes, load = scheduler.assign_nodes([0, 0, 0, 0], 100)
    assert np.bincount(nodes, minlength=4).tolist() == [25, 25, 25, 25]
    assert load.tolist() == [25, 25, 25, 25]
    assert nodes[:8].tolist() == [0, 1, 2, 3, 0, 1, 2, 3]              # round robin from idle


def test_greedy_fills_the_hole_first():
    nodes, load = scheduler.assign_nodes([5, 0, 3], 6)
    # 1 gets jobs until it reaches 3, then ties 1/2 alternate lowest id first
    assert nodes.tolist() == [1, 1, 1, 1, 2, 1] and load.tolist() == [5, 5, 4]


# ---------------------------------------------------------------- per-node batches

def test_spec_batches_drawn_from_own_queue():
    """interleaved arrivals across 2 nodes -> each batch only from its own queue."""
    pred = np.float32([400, 10, 30, 5, 200, 1])
    node = np.int32([0, 1, 0, 1, 0, 1])
    ids, cnt, pre, _ = scheduler.select_nodes(pred, [0] * 6, node, 2, 2)
    assert ids[0].tolist() == [2, 4] and ids[1].tolist() == [5, 3] and cnt.tolist() == [2, 2]
    assert not pre.any()


def test_node_not_ready_is_untouched():
    pred = np.float32([3, 2, 1, 9])
    node = np.int32([0, 1, 1, 0])
    running = np.uint8([1, 1, 0, 0])
    ids, cnt, pre, _ = scheduler.select_nodes(pred, [0] * 4, node, 2, 1, running=running,
                                              node_ready=[False, True])
    assert cnt.tolist() == [0, 1] and ids[0].tolist() == [-1] and ids[1].tolist() == [2]
    assert pre.tolist() == [0, 1, 0, 0]        # node 0's running job is mid-window, not preempted


@pytest.mark.parametrize("seed", range(10))
def test_select_nodes_invariants(seed):
    rng = np.random.default_rng(seed)
    n, W, cap = 300, 5, 7
    pred = rng.uniform(0, 100, n).astype(np.float32)
    gen = np.where(rng.random(n) < 0.1, -1, 0).astype(np.int32)
    node = rng.integers(0, W, n).astype(np.int32)
    order = rng.permutation(n).astype(np.uint32)
    ids, cnt, _, _ = scheduler.select_nodes(pred, gen, node, W, cap, order=order)
    for w in range(W):
        mine = [i for i in range(n) if node[i] == w and gen[i] >= 0]
        assert cnt[w] == min(cap, len(mine))
        sel = ids[w, :cnt[w]].tolist()
        assert all(node[i] == w for i in sel)
        key = {i: (float(pred[i]), int(order[i])) for i in mine}
        assert [key[i] for i in sel] == sorted(key[i] for i in sel)
        assert all(key[i] > key[sel[-1]] for i in mine if i not in sel)


# ---------------------------------------------------------------- starvation controls (f3)

def test_aging_closed_form():
    """key = max(0, rem - boost_amount * floor(waited / boost_after)): 100 - 10 * 3 = 70
    beats a fresh 75; a fresh 69 still wins over it."""
    ids, _, _, _ = isrtf_select(np.float32([100, 75]), [0, 0], 1, windows_waited=[6, 0],
                                boost_after=2, boost_amount=10.0)
    assert ids.tolist() == [0]
    ids, _, _, _ = isrtf_select(np.float32([100, 69]), [0, 0], 1, windows_waited=[7, 0],
                                boost_after=2, boost_amount=10.0)
    assert ids.tolist() == [1]


def test_aging_floor_at_zero_ties_by_order():
    ids, _, _, _ = isrtf_select(np.float32([10, 0.0]), [0, 0], 2, order=[1, 0], windows_waited=[10, 0],
                                boost_after=1, boost_amount=5.0)
    assert ids.tolist() == [1, 0]               # both keys 0 -> arrival rank decides


def test_preempt_margin():
    """A running job (remaining 100) keeps its slot against a newcomer predicted 95 with
    margin 10 (key 90 < 95) and loses to one predicted 85."""
    run = np.uint8([1, 0])
    ids, _, pre, _ = isrtf_select(np.float32([100, 95]), [50, 0], 1, running=run, preempt_margin=10.0)
    assert ids.tolist() == [0] and pre.tolist() == [0, 0]
    ids, _, pre, _ = isrtf_select(np.float32([100, 85]), [50, 0], 1, running=run, preempt_margin=10.0)
    assert ids.tolist() == [1] and pre.tolist() == [1, 0]


def test_aging_prevents_starvation():
    """One 500-token job at t = 0 and a 10-token job every 10 ms (cap 1, TPOT 1 ms, K = 50).
    Without aging the long job waits for the whole stream (first run at t = 1000); with aging
    (boost 50 per window waited) its key 500 - 50 w drops below 10 at w = 10 windows, so it
    first runs at the 11th batch, t = 100."""
    spec = [(0, 500)] + [(10 * k, 10) for k in range(100)]
    jobs = _jobs(spec)
    plain = scheduler.simulate_nodes(jobs, 1, POLICY_ISRTF, cap=1)
    assert plain[0][0] == 1000.0
    aged = scheduler.simulate_nodes(jobs, 1, POLICY_ISRTF, cap=1, boost_after=1, boost_amount=50.0)
    assert aged[0][0] == 100.0


# ---------------------------------------------------------------- multi-worker simulator

def test_two_workers_hand_example():
    """A (0, 100), B (0, 30), C (0, 20), 2 workers, cap 1: least-loaded sends A -> 0, B -> 1,
    C -> 0.  Node 0 runs C (0-20) then A (20-70-120); node 1 runs B (0-30)."""
    jobs = _jobs([(0, 100), (0, 30), (0, 20)])
    r = scheduler.simulate_nodes(jobs, 2, POLICY_ISRTF, cap=1)
    assert r[0] == (20.0, 120.0, 0) and r[1] == (0.0, 30.0, 1) and r[2] == (0.0, 20.0, 0)
    f = scheduler.simulate_nodes(jobs, 2, POLICY_FCFS, cap=1)
    assert f[0] == (0.0, 100.0, 0) and f[2] == (100.0, 120.0, 0)


def test_load_counts_finished_jobs():
    """A finishing job leaves its node's load: A (0, 10) on node 0 finishes at 10; B (0, 100) on
    node 1; C arriving at 10 (after A's window ended, event order (a) before (b)) goes to node 0."""
    jobs = _jobs([(0, 10), (0, 100), (10, 5)])
    r = scheduler.simulate_nodes(jobs, 2, POLICY_ISRTF, cap=1)
    assert r[2][2] == 0 and r[2][1] == 15.0


@pytest.mark.parametrize("seed", range(12))
def test_one_worker_equals_single_server_sim(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(5, 40))
    arr = np.sort(rng.integers(0, 400, n)).astype(float)
    tot = rng.integers(1, 300, n)
    jobs = [sim.SimJob(i, float(arr[i]), int(tot[i])) for i in range(n)]
    policy = [POLICY_ISRTF, POLICY_FCFS][seed % 2]
    cap = int(rng.integers(1, 5))
    allow = bool(seed % 3)
    a = sim.simulate(jobs, policy, cap=cap, ttft=3.0, tpot=1.5, allow_preempt=allow)
    b = scheduler.simulate_nodes(jobs, 1, policy, cap=cap, ttft=3.0, tpot=1.5, allow_preempt=allow)
    assert {k: v[:2] for k, v in b.items()} == a


def test_more_workers_never_hurt_fcfs_makespan():
    rng = np.random.default_rng(7)
    jobs = [sim.SimJob(i, float(10 * i), int(t)) for i, t in enumerate(rng.integers(20, 300, 40))]
    last = []
    for W in (1, 2, 4, 8):
        r = scheduler.simulate_nodes(jobs, W, POLICY_FCFS, cap=2)
        last.append(max(v[1] for v in r.values()))
    assert all(last[i + 1] <= last[i] for i in range(3))
