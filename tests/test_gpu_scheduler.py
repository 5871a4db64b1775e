"""Per-node Priority Buffers, least-loaded balancer and starvation controls on the B200
(SURVEY.md Sec. 8f rows f2, f3): bit-exact against oracle/scheduler.py and oracle/select.py
on identical fp32 predictions and integer states, through the C ABI (elis_assign_nodes,
elis_isrtf_select_nodes, elis_isrtf_select with elis_starvation)."""
import numpy as np
import pytest

from paper_2505_09142_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P(cuda_lib):
    from paper_2505_09142_b200 import binding
    cfg = inputs.CONFIGS["tiny"]
    p = binding.Predictor(cfg, inputs.flatten_weights(cfg, inputs.make_weights(cfg, seed=0)), 1024, 1024)
    yield p
    p.close()


def _d(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ---------------------------------------------------------------- load balancer

@pytest.mark.parametrize("W,n_new,seed", [(1, 5, 0), (2, 1, 1), (3, 7, 2), (4, 100, 3), (8, 1000, 4),
                                         (64, 5000, 5), (17, 0, 6), (5, 333, 7), (64, 3, 8)])
def test_assign_nodes_bit_exact(P, W, n_new, seed):
    from oracle.scheduler import assign_nodes
    rng = np.random.default_rng(seed)
    load = rng.integers(0, 50, W).astype(np.int32)
    if seed % 3 == 0:
        load[:] = 7                                  # all tied
    d_load = _d(load)
    out = torch.full((max(n_new, 1),), -9, dtype=torch.int32, device="cuda")
    P.assign_nodes(d_load, n_new, out)
    torch.cuda.synchronize()
    o_nodes, o_load = assign_nodes(load, n_new)
    np.testing.assert_array_equal(out.cpu().numpy()[:n_new], o_nodes)
    np.testing.assert_array_equal(d_load.cpu().numpy(), o_load)


def test_assign_nodes_spec_vectors(P):
    for load, want in (([3, 1, 2], 1), ([2, 2, 2], 0)):
        out = torch.empty(1, dtype=torch.int32, device="cuda")
        P.assign_nodes(_d(np.int32(load)), 1, out)
        assert int(out.item()) == want
    d_load = _d(np.zeros(4, np.int32))
    out = torch.empty(100, dtype=torch.int32, device="cuda")
    P.assign_nodes(d_load, 100, out)
    assert np.bincount(out.cpu().numpy(), minlength=4).tolist() == [25] * 4
    assert d_load.cpu().tolist() == [25] * 4


# ---------------------------------------------------------------- per-node select

def gpu_select_nodes(P, pred, gen, node, W, cap, policy, allow, order, running, ready, waited=None,
                     boost_after=1, boost_amount=0.0, margin=0.0):
    n = len(pred)
    ids = torch.full((W * cap,), -7, dtype=torch.int32, device="cuda")
    cnt = torch.full((W,), -7, dtype=torch.int32, device="cuda")
    pre = torch.full((max(n, 1),), 9, dtype=torch.uint8, device="cuda")
    P.isrtf_select_nodes(_d(pred), _d(gen), _d(node), W, cap, ids, cnt, node_ready=_d(ready), policy=policy,
                         allow_preempt=allow, order=_d(order), running=_d(running), out_preempted=pre,
                         windows_waited=_d(waited), boost_after=boost_after, boost_amount=boost_amount,
                         preempt_margin=margin)
    torch.cuda.synchronize()
    return ids.cpu().numpy().reshape(W, cap), cnt.cpu().numpy(), pre.cpu().numpy()[:n]


NODE_CASES = []
for seed in range(16):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.choice([1, 7, 100, 1000, 8192, 65536]))
    W = int(rng.choice([1, 2, 3, 8, 64]))
    cap = int(rng.choice([1, 4, 64, 256]))
    NODE_CASES.append((seed, n, W, cap))


@pytest.mark.parametrize("seed,n,W,cap", NODE_CASES)
def test_select_nodes_bit_exact(P, seed, n, W, cap):
    from oracle.scheduler import select_nodes
    rng = np.random.default_rng(seed)
    policy = int(rng.integers(0, 2))
    allow = bool(rng.integers(0, 2))
    pred = inputs.random_predictions(n, seed=seed, kind="mixed" if seed % 3 else "spread")
    gen, order, running = inputs.random_sched_state(n, seed=seed)
    node = rng.integers(0, W, n).astype(np.int32)
    ready = (rng.random(W) < 0.8).astype(np.uint8) if seed % 2 else None
    waited = rng.integers(0, 12, n).astype(np.int32) if seed % 4 == 1 else None
    amount = 25.0 if waited is not None else 0.0
    margin = float(rng.choice([0.0, 5.0, 40.0]))
    ids, cnt, pre = gpu_select_nodes(P, pred, gen, node, W, cap, policy, allow, order, running, ready,
                                     waited, 3, amount, margin)
    o_ids, o_cnt, o_pre, _ = select_nodes(pred, gen, node, W, cap, policy, allow, order, running,
                                          None if ready is None else ready.astype(bool), False, waited, 3,
                                          amount, margin)
    np.testing.assert_array_equal(cnt, o_cnt)
    np.testing.assert_array_equal(ids, o_ids)
    np.testing.assert_array_equal(pre, o_pre)


def test_select_nodes_spec_vector(P):
    """S:279 interleaved arrivals across 2 nodes -> each batch from its own queue."""
    pred = np.float32([400, 10, 30, 5, 200, 1])
    node = np.int32([0, 1, 0, 1, 0, 1])
    ids, cnt, pre = gpu_select_nodes(P, pred, np.zeros(6, np.int32), node, 2, 2, 0, True, None, None, None)
    assert ids.tolist() == [[2, 4], [5, 3]] and cnt.tolist() == [2, 2] and not pre.any()


def test_select_nodes_out_of_range_node_ignored(P):
    pred = np.float32([1, 2, 3])
    node = np.int32([0, 5, -1])
    running = np.uint8([0, 1, 1])
    ids, cnt, pre = gpu_select_nodes(P, pred, np.zeros(3, np.int32), node, 2, 2, 0, True, None, running, None)
    assert ids.tolist() == [[0, -1], [-1, -1]] and cnt.tolist() == [1, 0] and pre.tolist() == [0, 0, 0]


# ---------------------------------------------------------------- starvation controls on the single select

@pytest.mark.parametrize("seed", range(12))
def test_select_starvation_bit_exact(P, seed):
    from oracle.select import isrtf_select
    rng = np.random.default_rng(900 + seed)
    n = int(rng.choice([5, 300, 4096, 30000]))
    cap = int(rng.choice([1, 4, 64]))
    pred = inputs.random_predictions(n, seed=seed, kind="mixed")
    gen, order, running = inputs.random_sched_state(n, seed=seed, frac_running=0.3)
    waited = rng.integers(0, 40, n).astype(np.int32)
    after = int(rng.integers(1, 6))
    amount = float(rng.choice([0.0, 1.5, 10.0, 333.25]))
    margin = float(rng.choice([0.0, 0.5, 25.0]))
    allow = bool(seed % 3)
    ids = torch.full((cap,), -7, dtype=torch.int32, device="cuda")
    pre = torch.full((n,), 9, dtype=torch.uint8, device="cuda")
    cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    P.isrtf_select(_d(pred), _d(gen), cap, ids, allow_preempt=allow, order=_d(order), running=_d(running),
                   out_preempted=pre, out_count=cnt, windows_waited=_d(waited), boost_after=after,
                   boost_amount=amount, preempt_margin=margin)
    torch.cuda.synchronize()
    o_ids, o_cnt, o_pre, _ = isrtf_select(pred, gen, cap, 0, allow, order, running, False, waited, after,
                                          amount, margin)
    np.testing.assert_array_equal(ids.cpu().numpy(), o_ids)
    assert int(cnt.item()) == o_cnt
    np.testing.assert_array_equal(pre.cpu().numpy(), o_pre)


def test_starvation_rejects_bad_knobs(P):
    from paper_2505_09142_b200 import binding
    ids = torch.empty(1, dtype=torch.int32, device="cuda")
    z = _d(np.zeros(2, np.int32))
    with pytest.raises(binding.ElisError):
        P.isrtf_select(_d(np.float32([1, 2])), z, 1, ids, windows_waited=z, boost_after=0, boost_amount=1.0)
    with pytest.raises(binding.ElisError):
        P.isrtf_select(_d(np.float32([1, 2])), z, 1, ids, preempt_margin=-1.0)
